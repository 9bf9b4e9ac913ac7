"""N3 (hash-based dedup across GRPO rollouts, P:73 / P:271) on the GPU: vp_dedup_clips vs the oracle on random key
sequences (bit-exact ids and lists), and end to end -- the unique clips' rows, viewed per sample, are
byte-identical to processing every sample, and MRoPE over every sample's sequence from the per-sample grids equals
the oracle."""
import random

import numpy as np
import pytest
import torch

import oracle as O
import vp_inputs as I
from parity import host_frames, oracle_params, pack_frames

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(4))
def test_dedup_matches_oracle(seed):
    import paper_2604_16893_b200 as vp
    rng = random.Random(seed)
    for n in (0, 1, 7, 512, 1500, 3000):
        keys = [rng.randrange(max(1, n // rng.choice([1, 3, 8]))) * 0x9E3779B97F4A7C15 % (1 << 63) for _ in range(n)]
        k = torch.tensor(keys, dtype=torch.int64, device="cuda")
        uid = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        ul = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        nu = torch.empty(1, dtype=torch.int32, device="cuda")
        vp.dedup_clips(k, uid[:n], ul, nu)
        ref_id, ref_list = O.dedup_keys(keys)
        assert int(nu.item()) == len(ref_list)
        assert uid[:n].cpu().tolist() == ref_id and ul[: len(ref_list)].cpu().tolist() == ref_list


def test_grpo_batch_views_equal_full_processing():
    """16 samples = 4 prompts x 4 rollouts (mixed clip shapes, one image prompt): process the 4 unique clips,
    view them per sample, compare with processing all 16 samples (same frame bytes)."""
    import paper_2604_16893_b200 as vp
    pre = vp.VisualPreprocessor(max_frames=8, video_max_pixels=40000, image_max_pixels=65536, out_dtype=0)
    prompts = [I.clip(40, 10.0, 250, 500), I.clip(90, 30.0, 180, 320), I.image(300, 200), I.clip(12, 4.0, 64, 64)]
    samples = [prompts[i // 4] for i in range(16)]
    keys = [1000 + i // 4 for i in range(16)]
    uclips, ulist, uid = pre.dedup(samples, keys)
    assert ulist == [0, 4, 8, 12] and uid.cpu().tolist() == [i // 4 for i in range(16)]
    op = oracle_params(pre.params)
    # frames: identical bytes for the samples of one prompt (content seeded by the prompt)
    oplans, _ = O.plan_batch(op, samples)
    fl = [I.frames_u8("noise", i // 4, o.idx, o.in_h, o.in_w) for i, o in enumerate(oplans)]
    pit = [(3 * c["width"] + 15) // 16 * 16 for c in samples]
    buf, offs, pits = pack_frames(fl, pit)
    full = pre.run(pre.plan(samples), buf, offs, pits)
    upl = pre.plan(uclips)
    uout = pre.run(upl, buf, offs[ulist], pits[ulist])
    po, g, st = pre.views(upl, uid)
    torch.cuda.synchronize()
    fpl = pre.plan(samples)
    fph = fpl.plans_host
    for k in range(16):
        o = oplans[k]
        key = "pixel_values" if o.is_image else "pixel_values_videos"
        r0 = int(fph["patch_offset"][k])
        u0 = int(po[k])
        a = full[key][r0: r0 + o.patches].view(torch.int16)
        b = uout[key][u0: u0 + o.patches].view(torch.int16)
        assert torch.equal(a, b), k
        assert g[k].cpu().tolist() == list(o.grid)
    # MRoPE over every sample's sequence from the per-sample grids
    m = pre.params.merge_size
    seqs, ig, vg = [], [], []
    for o in oplans:
        if o.is_image:
            seqs.append(I.token_types([(0, 3), (1, o.tokens), (0, 2)]))
            ig.append(o.grid)
        else:
            runs = [(0, 4)]
            for _ in range(o.grid[0]):
                runs += [(0, 7), (2, o.grid[1] * o.grid[2] // m ** 2), (0, 1)]
            seqs.append(I.token_types(runs))
            vg.append(o.grid)
    isimg = torch.tensor([o.is_image for o in oplans], device="cuda", dtype=torch.bool)
    tt = torch.from_numpy(np.concatenate(seqs)).cuda()
    cu = torch.tensor(np.concatenate([[0], np.cumsum([len(s) for s in seqs])]), dtype=torch.int64).cuda()
    pos, deltas, _ = pre.rope_index(tt, cu, g[isimg], g[~isimg])
    ids, od, st2, bst = O.rope_index(seqs, ig, vg, m)
    assert np.array_equal(pos.cpu().numpy(), np.concatenate(ids, axis=1)) and deltas.cpu().tolist() == od
