"""GPU parity of K3 (vp_resize_normalize_patchify) against the f64 oracle (O4-O9).

Element-by-element on small/ragged batches (several tiles + ragged tails, odd T, images, identity,
up- and down-scale, misaligned pitches, fp32 and bf16), and on sampled outputs at the BASELINE
sizes in the bench's launch configuration.  Tolerances: fp32 1e-5 absolute; bf16 reading C15."""
import random

import numpy as np
import pytest
import torch

import oracle as O
import vp_inputs as I
from parity import assert_pixels, host_frames, oracle_params, pack_frames

pytestmark = pytest.mark.gpu


def _gpu_run(pre, clips, kind="noise", pitch_pad=0, frames=None, align16=False):
    pl = pre.plan(clips)
    op = oracle_params(pre.params)
    oplans, _ = O.plan_batch(op, clips)
    fl = host_frames(oplans, kind) if frames is None else frames
    # 16-B aligned pitches (and hence offsets) let the TMA variants take the clip; otherwise it is generic
    pitches = [(3 * c["width"] + 15) // 16 * 16 if align16 else 3 * c["width"] + pitch_pad for c in clips]
    buf, offs, pit = pack_frames(fl, pitches)
    out = pre.run(pl, buf, offs, pit)
    torch.cuda.synchronize()
    return pl, oplans, fl, out


def _full_compare(pre, clips, kind="noise", pitch_pad=0, align16=False):
    pl, oplans, fl, out = _gpu_run(pre, clips, kind, pitch_pad, align16=align16)
    op = oracle_params(pre.params)
    ref = O.process_batch(op, clips, [f if f is not None else np.zeros((1, 1, 1, 3), np.uint8) for f in fl],
                          plans=oplans)
    st = out["clip_status"][: len(clips)].cpu().numpy()
    assert st.tolist() == [p.status for p in oplans]
    assert out["image_grid_thw"].cpu().numpy().tolist() == ref["image_grid_thw"].tolist()
    assert out["video_grid_thw"].cpu().numpy().tolist() == ref["video_grid_thw"].tolist()
    assert_pixels(out["pixel_values"].cpu(), ref["pixel_values_images"], "images")
    assert_pixels(out["pixel_values_videos"].cpu(), ref["pixel_values_videos"], "videos")
    return out


@pytest.mark.parametrize("dtype", [1, 0])
def test_cfg1_full(dtype):
    import paper_2604_16893_b200 as vp
    params, clips = I.config("cfg1")
    params["out_dtype"] = dtype
    out = _full_compare(vp.VisualPreprocessor(**params), clips, kind="ramp")
    assert out["pixel_values_videos"].shape == (256, 1536)


@pytest.mark.parametrize("dtype", [1, 0])
def test_small_mixed_ragged_batch(dtype):
    """Videos and images, odd T (temporal pad), identity / down / up scale on either axis."""
    import paper_2604_16893_b200 as vp
    pre = vp.VisualPreprocessor(max_frames=7, video_max_pixels=64 * 96, image_max_pixels=96 * 128, out_dtype=dtype)
    clips = [I.clip(9, 2.0, 70, 100),          # n=7 (odd) -> pad; downscale
             I.image(64, 96),                  # identity image -> tp copies
             I.clip(3, 1.0, 20, 30),           # tiny -> upscale to 32x32
             I.image(150, 40),                 # down rows, up cols
             I.clip(6, 2.0, 64, 64),           # identity video (even n)
             I.clip(0, 30.0, 64, 64),          # invalid: skipped
             I.image(33, 257)]
    _full_compare(pre, clips)


@pytest.mark.parametrize("align16", [False, True])
@pytest.mark.parametrize("seed", range(4))
def test_random_shapes_and_pitches(seed, align16):
    """Random geometry and model params; unaligned pitches route clips to the generic kernel, 16-B aligned
    ones to the TMA fast / copy variants."""
    import paper_2604_16893_b200 as vp
    rng = random.Random(100 + seed)
    tp = rng.choice([1, 2, 3])
    pre = vp.VisualPreprocessor(max_frames=max(tp, rng.choice([2, 3, 5])), temporal_patch_size=tp,
                                patch_size=rng.choice([14, 16]), video_max_pixels=rng.choice([4096, 16384, 40000]),
                                image_max_pixels=rng.choice([16384, 65536]), out_dtype=rng.choice([0, 1]),
                                mean=(0.48145466, 0.4578275, 0.40821073), std=(0.26862954, 0.26130258, 0.27577711))
    clips = []
    for _ in range(rng.randint(1, 6)):
        h, w = rng.randint(8, 600), rng.randint(8, 600)
        clips.append(I.image(h, w) if rng.random() < 0.4 else I.clip(rng.randint(1, 40), rng.choice([2.0, 5.0]), h, w))
    _full_compare(pre, clips, pitch_pad=rng.choice([0, 1, 5, 16]), align16=align16)


@pytest.mark.parametrize("dtype", [1, 0])
def test_mild_upscale_and_identity_edges(dtype):
    """Ratios at the fast-path edges: in/out just above 0.8 (5-slot ring), identity, 1.0x-1.03x, and
    just below 0.8 (generic kernel)."""
    import paper_2604_16893_b200 as vp
    pre = vp.VisualPreprocessor(image_max_pixels=1048576, video_max_pixels=1048576, max_frames=3, out_dtype=dtype)
    clips = [I.image(27, 27), I.image(25, 25), I.image(1000, 1010), I.image(64, 96), I.clip(5, 2.0, 130, 100),
             I.image(820, 1000)]
    _full_compare(pre, clips)


@pytest.mark.parametrize("dtype", [1, 0])
@pytest.mark.parametrize("patch,tp", [(14, 3), (16, 2), (16, 1)])
def test_identity_copy_variant(dtype, patch, tp):
    """Both axes identity (KV_COPY): ragged merge-column chunks (gw/m = 11, 19), odd tp with temporal
    padding, images filling tp slots, a 1-frame video, and p = 14 (28-byte patch rows)."""
    import paper_2604_16893_b200 as vp
    f = 2 * patch
    pre = vp.VisualPreprocessor(patch_size=patch, temporal_patch_size=tp, max_frames=max(tp, 5),
                                image_max_pixels=f * f * 400, video_max_pixels=f * f * 400, out_dtype=dtype)
    clips = [I.image(2 * f, 11 * f), I.clip(5, 2.0, 3 * f, 19 * f), I.image(f, f), I.clip(1, 1.0, f, 2 * f),
             I.image(7 * f, 3 * f)]
    pl = pre.plan(clips)
    assert all(v == 4 for v in pl.plans_host["kernel_variant"][:len(clips)]), pl.plans_host["kernel_variant"]
    _full_compare(pre, clips)


def _aligned_compare(pre, clips, kind="noise"):
    """As _full_compare, with 16-B aligned row pitches (the TMA variants need them)."""
    pl = pre.plan(clips)
    op = oracle_params(pre.params)
    oplans, _ = O.plan_batch(op, clips)
    fl = host_frames(oplans, kind)
    buf, offs, pit = pack_frames(fl, [(3 * c["width"] + 15) // 16 * 16 for c in clips])
    out = pre.run(pl, buf, offs, pit)
    torch.cuda.synchronize()
    ref = O.process_batch(op, clips, [f if f is not None else np.zeros((1, 1, 1, 3), np.uint8) for f in fl],
                          plans=oplans)
    assert out["video_grid_thw"].cpu().numpy().tolist() == ref["video_grid_thw"].tolist()
    assert_pixels(out["pixel_values"].cpu(), ref["pixel_values_images"], "images")
    assert_pixels(out["pixel_values_videos"].cpu(), ref["pixel_values_videos"], "videos")
    return pl


CLIP_MEAN, CLIP_STD = (0.48145466, 0.4578275, 0.40821073), (0.26862954, 0.26130258, 0.27577711)


KV_TEAM, KV_WIDE = 5, 6


@pytest.mark.parametrize("dtype", [1, 0])
@pytest.mark.parametrize("tp", [1, 2, 3])
def test_team_variant(dtype, tp):
    """KV_TEAM (every warp does the 4-slot vertical ring and the horizontal pass of its column pairs): downscales
    from ~1.03x to ~2x, identity on one axis, several slices with a ragged last slice, temporal padding (n < tp and
    n not a multiple of tp), images filling tp slots, CLIP mean/std."""
    import paper_2604_16893_b200 as vp
    pre = vp.VisualPreprocessor(max_frames=max(tp, 5), temporal_patch_size=tp, video_max_pixels=32768,
                                image_max_pixels=65536, out_dtype=dtype, mean=CLIP_MEAN, std=CLIP_STD)
    clips = [I.clip(9, 2.0, 250, 500),        # 1.95x both axes -> 128 x 256
             I.image(64, 330),                # identity rows, 1.03x columns
             I.image(330, 64),                # 1.03x rows, identity columns
             I.clip(3, 1.0, 260, 1100),       # ~1.7x rows, ~2x columns: several slices
             I.clip(1, 1.0, 250, 500),        # n = 1 < tp: padded
             I.image(250, 500)]
    pl = _aligned_compare(pre, clips)
    kv = pl.plans_host["kernel_variant"][:len(clips)].tolist()
    assert sum(v in (KV_TEAM, KV_WIDE) for v in kv) >= 5, kv


@pytest.mark.parametrize("patch", [14, 16])
def test_team_patch14_and_wide(patch):
    """p = 14 (28-byte patch rows, slices in multiples of p) and a wide frame split into many slices."""
    import paper_2604_16893_b200 as vp
    f = 2 * patch
    pre = vp.VisualPreprocessor(patch_size=patch, max_frames=4, video_max_pixels=f * f * 300,
                                image_max_pixels=f * f * 300, out_dtype=1)
    clips = [I.clip(4, 1.0, 9 * f, 45 * f), I.image(12 * f + 5, 30 * f + 3), I.clip(2, 1.0, 500, 1000)]
    pl = _aligned_compare(pre, clips)
    assert np.isin(pl.plans_host["kernel_variant"][:len(clips)], (KV_TEAM, KV_WIDE)).all(), pl.plans_host["kernel_variant"]


@pytest.mark.parametrize("seed", range(3))
def test_team_random_downscales(seed):
    import paper_2604_16893_b200 as vp
    rng = random.Random(500 + seed)
    tp = rng.choice([1, 2])
    pre = vp.VisualPreprocessor(max_frames=rng.choice([2, 3, 4]), temporal_patch_size=tp,
                                video_max_pixels=rng.choice([16384, 40000, 90000]), image_max_pixels=65536,
                                out_dtype=rng.choice([0, 1]))
    clips = []
    for _ in range(rng.randint(2, 5)):
        h, w = rng.randint(40, 700), rng.randint(40, 700)
        clips.append(I.image(h, w) if rng.random() < 0.3 else I.clip(rng.randint(1, 9), 2.0, h, w))
    _aligned_compare(pre, clips)


def test_cfg2_one_clip_full():
    """BASELINE cfg2 at full size, compared element by element (64 frames 720p -> 384x672)."""
    import paper_2604_16893_b200 as vp
    params, clips = I.config("cfg2")
    params["out_dtype"] = 1
    _full_compare(vp.VisualPreprocessor(**params), clips)


def _sampled_compare(pre, clips, n_samples=4000, seed=0, kind="noise", align16=False):
    """Full-size launch; the oracle computes sampled outputs one by one (resize_pixel)."""
    pl, oplans, fl, out = _gpu_run(pre, clips, kind, align16=align16)
    op = oracle_params(pre.params)
    p, m, tp = op["patch_size"], op["merge_size"], op["temporal_patch_size"]
    rng = np.random.default_rng(seed)
    cache = {}
    for mod, key in ((True, "pixel_values"), (False, "pixel_values_videos")):
        pv = out[key]
        sel = [o for o in oplans if o.status == O.VP_OK and o.is_image == mod]
        if not sel:
            continue
        got_rows, ref_vals, gpu_vals = [], [], []
        for _ in range(n_samples):
            o = sel[rng.integers(len(sel))]
            r = int(rng.integers(o.patches))
            q = int(rng.integers(pv.shape[1]))
            slot, y, x, c = O.patch_coords(r, q, o.grid, p, m, tp)
            k = oplans.index(o)
            fr = fl[k][min(slot, o.n - 1)]
            v = O.resize_pixel(fr, o.out_h, o.out_w, y, x, c, cache)
            ref_vals.append((v / 255.0 - op["mean"][c]) / op["std"][c])
            got_rows.append((o.patch_offset + r, q))
        idx = torch.tensor(got_rows, dtype=torch.int64, device=pv.device)
        g = pv[idx[:, 0], idx[:, 1]].cpu()
        assert_pixels(g, np.array(ref_vals), key)


def test_cfg3_sampled():
    import paper_2604_16893_b200 as vp
    params, clips = I.config("cfg3")
    _sampled_compare(vp.VisualPreprocessor(**params), clips, n_samples=3000)


def test_cfg4_sampled():
    import paper_2604_16893_b200 as vp
    params, clips = I.config("cfg4")
    _sampled_compare(vp.VisualPreprocessor(**params), clips, n_samples=3000)


def test_fast_groups_straddle_items():
    """The TMA staging of the team / fast kernels refills in groups of 8 source rows; when a source height is
    not a multiple of 8 a group straddles two work items (the per-row refill path that opens the next item).
    40 odd-height clips x 16 frames (x slices) over the whole GPU, so every CTA walks several consecutive items
    of different heights and geometries (distinct weight tables); sampled outputs of every clip vs the oracle."""
    import paper_2604_16893_b200 as vp
    rng = random.Random(7)
    pre = vp.VisualPreprocessor(max_frames=16, video_max_pixels=100000, out_dtype=1)   # ratios ~1.1-2.1
    clips = []
    while len(clips) < 40:
        h, w = rng.randint(300, 520), rng.randint(380, 700)
        if h % 8:
            clips.append(I.clip(240, 30.0, h, w))
    kv = pre.plan(clips).plans_host["kernel_variant"][:len(clips)]
    assert all(v in (0, 1, 2, KV_TEAM, KV_WIDE) for v in kv) and sum(v in (KV_TEAM, KV_WIDE) for v in kv) >= 30, kv
    _sampled_compare(pre, clips, n_samples=6000, seed=3, align16=True)


def test_cfg5_bench_launch_sampled():
    """The bench's own workload and launch configuration (bench.py cfg5): 512 full-size cfg2 clips (90.6 GB of
    device-synthesised noise frames, seed = clip index, as bench.py), bf16 output, one K3 call over the whole
    batch; 16 (clip, source frame) pairs x 128 sampled outputs are recomputed one by one by the oracle from
    the host twin of the frame generator."""
    import paper_2604_16893_b200 as vp
    params = I.qwen3_params(max_frames=64)
    clips = [I.clip(1800, 30.0, 720, 1280)] * 512
    pre = vp.VisualPreprocessor(**params)
    pl = pre.plan(clips)
    ph = pl.plans_host
    off, pitch, total = pre.frames_layout(pl)
    frames = torch.empty(total, dtype=torch.uint8, device="cuda")
    idx_host = pl.frame_indices.cpu().numpy()
    for k in range(len(clips)):
        n = int(ph["n_frames"][k])
        ids = torch.from_numpy(idx_host[ph["index_offset"][k]: ph["index_offset"][k] + n].copy()).cuda()
        vp.synth_frames(vp.VP_SYNTH_NOISE, k, ids, 720, 1280, frames[off[k]:], int(pitch[k]))
    out = pre.run(pl, frames, torch.from_numpy(off).cuda(), torch.from_numpy(pitch).cuda(), strict=True)
    torch.cuda.synchronize()
    del frames
    op = oracle_params(pre.params)
    oplans, _ = O.plan_batch(op, clips[:1])
    o = oplans[0]
    p, m, tp = op["patch_size"], op["merge_size"], op["temporal_patch_size"]
    pv = out["pixel_values_videos"]
    rng = np.random.default_rng(5)
    rows, ref = [], []
    per_clip_rows = o.patches
    for k in rng.choice(len(clips), 16, replace=False):
        k = int(k)
        f = int(rng.integers(o.n))                      # a sampled source frame of clip k
        fid = int(idx_host[ph["index_offset"][k] + f])
        fr = I.frames_u8("noise", k, [fid], 720, 1280)[0]
        cache = {}
        got = 0
        while got < 128:
            r, q = int(rng.integers(per_clip_rows)), int(rng.integers(pv.shape[1]))
            slot, y, x, c = O.patch_coords(r, q, o.grid, p, m, tp)
            if min(slot, o.n - 1) != f:
                continue
            v = O.resize_pixel(fr, o.out_h, o.out_w, y, x, c, cache)
            ref.append((v / 255.0 - op["mean"][c]) / op["std"][c])
            rows.append((int(ph["patch_offset"][k]) + r, q))
            got += 1
    idx = torch.tensor(rows, dtype=torch.int64, device=pv.device)
    assert_pixels(pv[idx[:, 0], idx[:, 1]].cpu(), np.array(ref), "cfg5 videos")
    assert out["video_grid_thw"].cpu().tolist() == [[32, 24, 42]] * 512
    # every one of the 49.5 M bf16 values of the first and the last clip of the launch, element by element
    for k in (0, len(clips) - 1):
        fr = I.frames_u8("noise", k, o.idx, 720, 1280)
        refk = O.process_batch(op, clips[:1], [fr], plans=oplans)["pixel_values_videos"]
        r0 = int(ph["patch_offset"][k])
        assert_pixels(pv[r0: r0 + o.patches].cpu(), refk, f"cfg5 clip {k} (all values)")
        del refk


def test_cfg5_rank_shards_byte_identical():
    """Rank-count independence (the S:150 worker-count-independence analogue for clip sharding, DESIGN.md section
    7): the 512-clip cfg5 job run as one call and as the shards ranks of a world of 2 / 8 / 64 would run -- each
    shard planned on its own (offsets from 0) over the same frame bytes -- gives byte-identical rows."""
    import paper_2604_16893_b200 as vp
    params = I.qwen3_params(max_frames=64)
    clips = [I.clip(1800, 30.0, 720, 1280)] * 512
    pre = vp.VisualPreprocessor(**params)
    pl = pre.plan(clips)
    ph = pl.plans_host
    off, pitch, total = pre.frames_layout(pl)
    frames = torch.empty(total, dtype=torch.uint8, device="cuda")
    idx_host = pl.frame_indices.cpu().numpy()
    for k in range(len(clips)):
        n = int(ph["n_frames"][k])
        ids = torch.from_numpy(idx_host[ph["index_offset"][k]: ph["index_offset"][k] + n].copy()).cuda()
        vp.synth_frames(vp.VP_SYNTH_NOISE, k, ids, 720, 1280, frames[off[k]:], int(pitch[k]))
    offd, pitd = torch.from_numpy(off).cuda(), torch.from_numpy(pitch).cuda()
    whole = pre.run(pl, frames, offd, pitd, strict=True)["pixel_values_videos"]
    for a, b in ((256, 264), (448, 512), (504, 512), (0, 8)):       # shards of world 64/8/64 and rank 0
        sp = pre.plan(clips[a:b])
        part = pre.run(sp, frames, offd[a:b], pitd[a:b], strict=True)["pixel_values_videos"]
        r0 = int(ph["patch_offset"][a])
        assert torch.equal(part.view(torch.int16), whole[r0: r0 + part.shape[0]].view(torch.int16)), (a, b)


def test_determinism_three_runs():
    """AC12: three runs are byte-identical."""
    import paper_2604_16893_b200 as vp
    params, clips = I.config("cfg4")
    clips = clips[14:18]
    pre = vp.VisualPreprocessor(**params)
    outs = [_gpu_run(pre, clips)[3] for _ in range(3)]
    for o in outs[1:]:
        for k in ("pixel_values", "pixel_values_videos"):
            assert torch.equal(o[k].view(torch.int16), outs[0][k].view(torch.int16))


def test_capacity_is_reported_not_overrun():
    import paper_2604_16893_b200 as vp
    params, clips = I.config("cfg1")
    pre = vp.VisualPreprocessor(**params)
    pl = pre.plan(clips)
    out = pre.alloc_outputs(pl)
    big = torch.full((300, 1536), 7.0, dtype=torch.bfloat16, device="cuda")
    out["pixel_values_videos"] = big[:100]               # needs 256 rows
    fl = host_frames(O.plan_batch(oracle_params(pre.params), clips)[0])
    buf, offs, pit = pack_frames(fl, [384])
    pre.run(pl, buf, offs, pit, out=out, strict=False)
    assert out["clip_status"][0].item() == vp.VP_ECAPACITY
    with pytest.raises(vp.VpError):
        pre.run(pl, buf, offs, pit, out=out)                  # strict by default
    assert (big.float() == 7.0).all()


def test_synth_frames_match_host_generator():
    import paper_2604_16893_b200 as vp
    for kind, kid in (("ramp", vp.VP_SYNTH_RAMP), ("noise", vp.VP_SYNTH_NOISE)):
        ids = [3, 17, 1799]
        H, W, pitch = 37, 53, 3 * 53 + 7
        out = torch.zeros(len(ids) * H * pitch, dtype=torch.uint8, device="cuda")
        vp.synth_frames(kid, 12345, torch.tensor(ids, device="cuda"), H, W, out, row_pitch=pitch)
        got = out.cpu().numpy().reshape(len(ids), H, pitch)[:, :, : 3 * W].reshape(len(ids), H, W, 3)
        assert np.array_equal(got, I.frames_u8(kind, 12345, ids, H, W))


KV_TEAML = 8


@pytest.mark.parametrize("dtype", [0, 1])
def test_team_large_downscales(dtype):
    """KV_TEAML (the team kernel with unswizzled, padded retire rows and <= 32-tap column-pair windows): 1440p and
    2160p sources at the cfg2 video budget (3.75x / 5.6x), 1200 source rows at a small budget, an odd frame count, next to a
    cfg2-ratio clip (KV_WIDE) in the same call; every element vs the oracle."""
    import paper_2604_16893_b200 as vp
    pre = vp.VisualPreprocessor(max_frames=3, video_max_pixels=262144, out_dtype=dtype, mean=CLIP_MEAN, std=CLIP_STD)
    clips = [I.clip(3, 1.0, 1440, 2560), I.clip(1, 1.0, 2160, 3840), I.clip(3, 1.0, 720, 1280)]
    pl = _aligned_compare(pre, clips)
    kv = pl.plans_host["kernel_variant"][: len(clips)].tolist()
    assert kv[0] == KV_TEAML and kv[1] == KV_TEAML and kv[2] == KV_WIDE, kv
    pre2 = vp.VisualPreprocessor(max_frames=2, video_max_pixels=65536, out_dtype=dtype)
    pl2 = _aligned_compare(pre2, [I.clip(2, 1.0, 1200, 1920), I.clip(2, 1.0, 1080, 1920)])
    kv2 = pl2.plans_host["kernel_variant"][:2].tolist()
    assert kv2[0] == KV_TEAML and kv2[1] in (0, 1, 2), kv2      # <= 1088 source rows: the fast streaming kernel


@pytest.mark.parametrize("patch,merge,tp", [(6, 1, 1), (16, 2, 2), (14, 2, 2)])
def test_team_row_bands(patch, merge, tp):
    """Launches too small to fill the GPU cut each frame into row bands (one item per band, halo source rows shared
    with the neighbours, rows of the band above accumulated and dropped): a single 720p clip and a two-clip batch
    (KV_WIDE), a wide clip (KV_TEAM slices x bands) and a 1440p clip (KV_TEAML); non-preset geometry (p = 6, m = 1:
    output heights not a multiple of 4) takes the dynamic retire-slot path.  Every element vs the oracle, and the
    banded single-clip call byte-identical to the same clip inside a large (unbanded) batch."""
    import paper_2604_16893_b200 as vp
    f = patch * merge
    pre = vp.VisualPreprocessor(patch_size=patch, merge_size=merge, temporal_patch_size=tp, max_frames=4,
                                video_max_pixels=f * f * 160, image_max_pixels=f * f * 160, out_dtype=1)
    _aligned_compare(pre, [I.clip(4, 1.0, 720, 1280)])
    _aligned_compare(pre, [I.clip(3, 1.0, 720, 1280), I.clip(2, 1.0, 500, 900)])
    _aligned_compare(pre, [I.clip(2, 1.0, 600, 2000)])
    _aligned_compare(pre, [I.clip(2, 1.0, 1440, 2560)])
    # byte identity: the clip alone (banded) vs the same clip first in a 150-clip batch (600 items: whole frames)
    one = [I.clip(4, 1.0, 720, 1280)]
    many = one * 150
    op = oracle_params(pre.params)
    fr = host_frames(O.plan_batch(op, one)[0], "noise")
    _, _, _, out1 = _gpu_run(pre, one, frames=fr, align16=True)
    _, _, _, out2 = _gpu_run(pre, many, frames=fr * 150, align16=True)
    rows = int(out1["pixel_values_videos"].shape[0])
    assert rows > 0
    assert torch.equal(out1["pixel_values_videos"][:rows].view(torch.int16),
                       out2["pixel_values_videos"][:rows].view(torch.int16))
