"""GPU parity of K1 (vp_plan_frames): plans, frame indices, timestamps and totals are bit-exact
against the oracle (O1-O3, O10, H4) over random and edge-case clip sets."""
import random

import numpy as np
import pytest
import torch

import oracle as O
import vp_inputs as I

pytestmark = pytest.mark.gpu


def _run(params_kw, clips):
    import paper_2604_16893_b200 as vp
    pre = vp.VisualPreprocessor(**params_kw)
    pl = pre.plan(clips)
    return pre, pl


def _compare(params_kw, clips):
    import paper_2604_16893_b200 as vp
    pre, pl = _run(params_kw, clips)
    from parity import oracle_params
    op = oracle_params(pre.params)
    oplans, otot = O.plan_batch(op, clips)
    ph = pl.plans_host
    idx = pl.frame_indices.cpu().numpy()
    ts = pl.group_timestamps.cpu().numpy()
    for k, (o, c) in enumerate(zip(oplans, clips)):
        g = ph[k]
        assert g["status"] == o.status, (k, c)
        assert g["is_image"] == int(o.is_image)
        if o.status != O.VP_OK:
            continue
        got = (g["n_frames"], g["out_h"], g["out_w"], g["grid_t"], g["grid_h"], g["grid_w"])
        assert got == (o.n, o.out_h, o.out_w) + tuple(o.grid), (k, c, got)
        assert (g["index_offset"], g["patch_offset"], g["token_offset"], g["grid_index"]) == (
            o.index_offset, o.patch_offset, o.token_offset, o.grid_index), k
        assert idx[o.index_offset: o.index_offset + o.n].tolist() == o.idx, k
        if not o.is_image:
            assert g["group_offset"] == o.group_offset
            assert g["effective_fps"] == o.eff_fps                       # bit-exact f64
            ots = O.group_timestamps(o.idx, c["source_fps"], op["temporal_patch_size"])
            assert ts[o.group_offset: o.group_offset + len(ots)].tolist() == ots, k   # bit-exact f64
    t = pl.totals
    assert t["indices"] == otot["indices"]
    for key in ("img_rows", "vid_rows", "img_tokens", "vid_tokens", "n_images", "n_videos"):
        assert t[key] == otot[key], key
    assert t["vid_groups"] == otot["vid_groups"] and t["flags"] == 0
    assert t["n_invalid"] == sum(o.status != O.VP_OK for o in oplans)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_plan_baseline_configs(name):
    params, clips = I.config(name)
    kw = {k: v for k, v in params.items()}
    _compare(kw, clips)


def _random_clips(rng, n):
    clips = []
    for _ in range(n):
        r = rng.random()
        if r < 0.3:
            clips.append(I.image(rng.randint(1, 4000), rng.randint(1, 4000)))
        elif r < 0.35:   # invalid descriptors
            clips.append(I.clip(rng.choice([0, -5, 10]), rng.choice([0.0, -1.0, 30.0]) if rng.random() < .5 else 0.0,
                                rng.randint(1, 99), rng.randint(1, 99)))
        else:
            clips.append(I.clip(rng.choice([1, 2, 3, 7, rng.randint(1, 200000)]),
                                rng.choice([1.0, 23.976, 24.0, 25.0, 29.97, 30.0, 60.0, rng.uniform(0.2, 240.0)]),
                                rng.randint(1, 4000), rng.randint(1, 4000)))
    return clips


@pytest.mark.parametrize("seed", range(6))
def test_plan_random_batches(seed):
    rng = random.Random(seed)
    kw = dict(target_fps=rng.choice([0.5, 1.0, 2.0, 4.0]), max_frames=rng.choice([2, 16, 64, 128, 768]),
              temporal_patch_size=rng.choice([1, 2, 3]), patch_size=rng.choice([14, 16]), merge_size=2,
              video_max_pixels=rng.choice([262144, 100352, 1048576]), image_max_pixels=rng.choice([1048576, 200704]),
              min_pixels=rng.choice([0, 3136, 16384]), budget_mode=rng.choice([0, 1]))
    if kw["budget_mode"] == 1:
        kw["video_max_pixels"] = rng.choice([25165824, 12845056])
    kw["max_frames"] = max(kw["max_frames"], kw["temporal_patch_size"])
    _compare(kw, _random_clips(rng, rng.choice([1, 37, 600, 1500])))


def test_plan_empty_and_overflow_flags():
    import paper_2604_16893_b200 as vp
    pre = vp.VisualPreprocessor()
    pl = pre.plan([])
    assert pl.totals["indices"] == 0 and pl.totals["tiles"] == 0
    # undersized index buffer -> flag, no out-of-bounds write
    desc = torch.from_numpy(vp.clip_desc_array([I.clip(1800, 30.0, 720, 1280)]).view(np.uint8)).cuda()
    plans = torch.empty(vp.PLAN_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    idx = torch.full((10,), -7, dtype=torch.int64, device="cuda")
    tot = torch.empty(vp.TOT_LEN, dtype=torch.int64, device="cuda")
    vp.plan_frames(pre.params, desc, 1, plans, idx, tot)
    assert tot[vp.TOT["flags"]].item() & 1
    assert (idx.cpu() >= 0).all()


@pytest.mark.parametrize("seed", range(4))
def test_plan_hf_linspace_sampling(seed):
    """N1 sampling (VP_SAMPLE_LINSPACE, HF Qwen3-VL sample_frames): n, indices, effective fps and timestamps
    bit-exact vs the oracle (itself pinned to HF in tests/test_oracle_plan.py), incl. n not a multiple of tp
    (temporal pad), n < min_frames clamps, total < min_frames, and min_frames = 0 with sub-frame durations."""
    rng = random.Random(40 + seed)
    kw = dict(target_fps=rng.choice([0.5, 1.0, 2.0, 4.0]), max_frames=rng.choice([16, 64, 768]),
              temporal_patch_size=rng.choice([1, 2, 3]), patch_size=16, merge_size=2,
              video_max_pixels=262144, image_max_pixels=1048576, sampling=1, min_frames=rng.choice([0, 1, 4]))
    _compare(kw, _random_clips(rng, rng.choice([37, 600, 1500])))
