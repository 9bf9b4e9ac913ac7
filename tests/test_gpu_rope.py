"""GPU parity of K4 (vp_rope_index) against the oracle (O11): ids and deltas bit-exact, strict
validation statuses identical, over the mixed cfg4-shaped batch, an LVBench-length sequence, the
classic / time-scaled variants, and a fuzz of sequences with adversarial off-by-one runs."""
import random

import numpy as np
import pytest
import torch

import oracle as O
import vp_inputs as I

pytestmark = pytest.mark.gpu


def _gpu_rope(seqs, img, vid, m, variant=0, spg=None, tps=0):
    import paper_2604_16893_b200 as vp
    pre = vp.VisualPreprocessor(merge_size=m)
    tt = torch.from_numpy(np.concatenate(seqs).astype(np.int8) if seqs else np.zeros(0, np.int8)).cuda()
    cu = torch.tensor(np.concatenate([[0], np.cumsum([len(s) for s in seqs])]), dtype=torch.int64).cuda()
    ig = torch.tensor(img, dtype=torch.int64).reshape(-1, 3).cuda() if img else None
    vg = torch.tensor(vid, dtype=torch.int64).reshape(-1, 3).cuda() if vid else None
    sp = torch.tensor(spg, dtype=torch.float64).cuda() if spg is not None else None
    pos, deltas, st = pre.rope_index(tt, cu, ig, vg, variant=variant, second_per_grid=sp, tokens_per_second=tps,
                                     strict=False)
    torch.cuda.synchronize()
    return pos.cpu().numpy(), deltas.cpu().numpy(), st.cpu().numpy()


def _compare(seqs, img, vid, m, variant=0, spg=None, tps=0):
    ids, deltas, st, bst = O.rope_index(seqs, img, vid, m, variant=variant, second_per_grid_ts=spg,
                                        tokens_per_second=tps)
    pos, gd, gst = _gpu_rope(seqs, img, vid, m, variant, spg, tps)
    assert gst[:-1].tolist() == st and gst[-1] == bst
    off = 0
    for b, (s, a) in enumerate(zip(seqs, ids)):
        if st[b] == O.VP_OK:
            assert np.array_equal(pos[:, off: off + len(s)], a), b
            assert gd[b] == deltas[b], b
        off += len(s)
    return st, bst


def _video_runs(grid, m, ts_len=6):
    t, h, w = grid
    runs = []
    for _ in range(t):
        runs += [(0, ts_len + 1), (2, h * w // m ** 2), (0, 1)]
    return runs


def test_cfg4_shaped_batch():
    """16 image sequences (1,64,64) + 8 video sequences (32,24,42) + one interleaved sequence."""
    m = 2
    img, vid, seqs = [], [], []
    for _ in range(16):
        img.append((1, 64, 64))
        seqs.append(I.token_types([(0, 64), (0, 1), (1, 1024), (0, 1), (0, 32)]))
    for _ in range(8):
        vid.append((32, 24, 42))
        seqs.append(I.token_types([(0, 64)] + _video_runs((32, 24, 42), m) + [(0, 32)]))
    img += [(1, 32, 48), (1, 16, 16)]
    vid.append((3, 16, 32))
    seqs.append(I.token_types([(0, 5), (1, 384), (0, 3)] + _video_runs((3, 16, 32), m) + [(0, 2), (1, 64), (0, 9)]))
    st, bst = _compare(seqs, img, vid, m)
    assert all(s == O.VP_OK for s in st) and bst == O.VP_OK


def test_lvbench_long_sequence():
    """cfg3: 384 groups of (1,8,14) -> 10,752 visual tokens + timestamps in one sequence."""
    m = 2
    seq = I.token_types([(0, 100)] + _video_runs((384, 8, 14), m) + [(0, 50)])
    st, _ = _compare([seq], [], [(384, 8, 14)], m)
    assert st == [O.VP_OK]


def test_classic_and_time_scaled_variants():
    m = 2
    vid = [(3, 4, 4), (2, 8, 6), (5, 2, 2)]
    seqs = [I.token_types([(0, 4), (2, 12), (0, 3)]), I.token_types([(0, 1), (2, 24), (0, 2), (2, 5), (0, 1)])]
    _compare(seqs, [], vid, m, variant=1)
    _compare(seqs, [], vid, m, variant=2, spg=[1.0, 2.5, 4.0], tps=25)
    _compare(seqs, [], vid, m, variant=2, spg=[2 / 0.7, 2 / 3.0, 2.0], tps=13)   # truncation, interval 0


def test_text_only_and_empty():
    _compare([np.zeros(1000, np.int8), np.zeros(0, np.int8), np.zeros(1, np.int8)], [], [], 2)
    pos, d, st = _gpu_rope([], [(1, 4, 4)], [], 2)
    assert st[-1] == O.VP_EMISMATCH          # leftover grid, no sequences


@pytest.mark.parametrize("seed", range(3))
def test_fuzz_with_adversarial_mismatches(seed):
    """S:662 AC9-style fuzz: random batches where some runs are off by one or glued together."""
    rng = random.Random(seed)
    m = 2
    for _ in range(30):
        img, vid, seqs = [], [], []
        for _ in range(rng.randint(1, 40)):
            runs = [(0, rng.randint(0, 20))]
            for _ in range(rng.randint(0, 4)):
                if rng.random() < 0.5:
                    g = (1, 2 * rng.randint(1, 12), 2 * rng.randint(1, 12))
                    img.append(g)
                    n = g[1] * g[2] // 4
                    if rng.random() < 0.1:
                        n += rng.choice([-1, 1])
                    runs += [(1, max(n, 1)), (0, rng.randint(1, 5))]
                else:
                    g = (rng.randint(1, 5), 2 * rng.randint(1, 8), 2 * rng.randint(1, 8))
                    vid.append(g)
                    for gi in range(g[0]):
                        n = g[1] * g[2] // 4
                        if rng.random() < 0.05:
                            n += rng.choice([-1, 1])
                        runs += [(0, rng.randint(1, 4)) if (gi == 0 or rng.random() > 0.03) else (0, 0),
                                 (2, max(n, 1))]
                    runs.append((0, rng.randint(1, 3)))
            runs = [r for r in runs if r[1] > 0]
            seqs.append(I.token_types(runs))
        if rng.random() < 0.1 and img:
            img.pop()                                        # a run without a grid
        _compare(seqs, img, vid, m)


@pytest.mark.parametrize("name", ["qwen2_vl", "qwen2_5_vl", "qwen3_vl", "qwen3_5"])
def test_presets_end_to_end(name):
    """N2: each family preset through plan -> (Qwen2.5: vp_plan_second_per_grid) -> MRoPE, vs the oracle; the
    per-video seconds per grid bit-exact with the oracle's HF-order sampled fps."""
    import paper_2604_16893_b200 as vp
    pre = vp.VisualPreprocessor.from_preset(name, max_frames=16, video_max_pixels=50176)
    clips = [I.clip(300, 29.97, 360, 640), I.image(300, 400), I.clip(50, 10.0, 224, 224), I.clip(7, 2.0, 100, 90),
             I.clip(1000, 59.94, 480, 854)]
    pl = pre.plan(clips)
    from parity import oracle_params
    op = oracle_params(pre.params)
    oplans, _ = O.plan_batch(op, clips)
    m = op["merge_size"]
    spg = pre.second_per_grid(pl).cpu().tolist()
    ref_spg = [O.second_per_grid(op["temporal_patch_size"], O.hf_sampled_fps(o.n, c["total_source_frames"],
                                                                             c["source_fps"]))
               for o, c in zip(oplans, clips) if not o.is_image]
    assert spg == ref_spg
    seqs, ig, vg = [], [], []
    for o in oplans:
        if o.is_image:
            seqs.append(I.token_types([(0, 3), (1, o.tokens), (0, 2)]))
            ig.append(o.grid)
        else:
            vg.append(o.grid)
            if pre.rope_variant == vp.VP_ROPE_QWEN3_SPLIT:
                runs = [(0, 4)]
                for _ in range(o.grid[0]):
                    runs += [(0, 7), (2, o.grid[1] * o.grid[2] // m ** 2), (0, 1)]
            else:
                runs = [(0, 4), (2, o.tokens), (0, 3)]
            seqs.append(I.token_types(runs))
    tt = torch.from_numpy(np.concatenate(seqs)).cuda()
    cu = torch.tensor(np.concatenate([[0], np.cumsum([len(s) for s in seqs])]), dtype=torch.int64).cuda()
    igt = torch.tensor(ig, dtype=torch.int64).cuda()
    vgt = torch.tensor(vg, dtype=torch.int64).cuda()
    pos, deltas, st = pre.rope_index(tt, cu, igt, vgt, second_per_grid=pre.second_per_grid(pl))
    ids, od, ost, bst = O.rope_index(seqs, ig, vg, m, variant=pre.rope_variant, second_per_grid_ts=ref_spg,
                                     tokens_per_second=pre.tokens_per_second)
    assert np.array_equal(pos.cpu().numpy(), np.concatenate(ids, axis=1)) and deltas.cpu().tolist() == od


def test_ac9_strict_alignment_fuzz_10000_batches():
    """S:662 AC9 at its stated scale: 10,000 random batches (1-6 sequences of text / image / video runs) with
    adversarial off-by-one runs, glued video groups and missing grids; statuses, ids and deltas vs the oracle.
    Batches are concatenated 100 at a time into one packed call (sequence statuses are per sequence; the batch
    status is checked per call)."""
    rng = random.Random(9000)
    m = 2
    checked = 0
    for call in range(100):
        img, vid, seqs = [], [], []
        for _ in range(100):                             # 100 batches of 1-6 sequences per packed call
            for _ in range(rng.randint(1, 6)):
                runs = [(0, rng.randint(0, 6))]
                for _ in range(rng.randint(0, 3)):
                    if rng.random() < 0.5:
                        g = (1, 2 * rng.randint(1, 6), 2 * rng.randint(1, 6))
                        img.append(g)
                        n = g[1] * g[2] // 4 + (rng.choice([-1, 1]) if rng.random() < 0.15 else 0)
                        runs += [(1, max(n, 1)), (0, rng.randint(1, 3))]
                    else:
                        g = (rng.randint(1, 3), 2 * rng.randint(1, 4), 2 * rng.randint(1, 4))
                        vid.append(g)
                        for gi in range(g[0]):
                            n = g[1] * g[2] // 4 + (rng.choice([-1, 1]) if rng.random() < 0.08 else 0)
                            runs += [(0, rng.randint(1, 3)) if (gi == 0 or rng.random() > 0.05) else (0, 0),
                                     (2, max(n, 1))]
                        runs.append((0, rng.randint(1, 2)))
                runs = [r for r in runs if r[1] > 0]
                seqs.append(I.token_types(runs))
            checked += 1
        if rng.random() < 0.2 and img:
            img.pop()
        _compare(seqs, img, vid, m)
    assert checked == 10000
