"""Pins for oracle O1-O3 (frame plan, smart_resize, grid) against things other than itself:
SPEC worked examples (tests/golden), exact rational arithmetic, closed-form bounds,
HF transformers' smart_resize (library pin, reading C6), brute-force invariants."""
import math
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import vp_inputs as I


# ---------------- O1 frame plan ----------------

def test_spec_sampling_examples(golden):
    ex = golden["sample_frame_indices"]
    e = ex[0]
    n, idx = O.sample_frame_indices(e["total"], e["source_fps"], e["target_fps"], e["max_frames"], e["tp"])
    assert n == e["n"]
    assert idx[:3] == e["indices_head"] and idx[-1] == e["indices_last"]
    assert all(b - a == e["indices_step"] for a, b in zip(idx, idx[1:]))
    e = ex[1]
    assert O.sample_frame_indices(e["total"], e["source_fps"], e["target_fps"], e["max_frames"], e["tp"]) == (
        e["n"], e["indices"])
    e = ex[2]
    total = int(e["duration_s"] * e["source_fps"])
    n, _ = O.sample_frame_indices(total, e["source_fps"], e["target_fps"], e["max_frames"], e["tp"])
    assert n == e["n"]


def test_sampling_invalid_inputs():
    for total, fps in [(0, 30.0), (-3, 30.0), (10, 0.0), (10, -1.0)]:
        with pytest.raises(ValueError):
            O.sample_frame_indices(total, fps, 2.0, 64, 2)


def test_center_of_bin_matches_exact_rational():
    """S:78 floor((i+0.5)*total/n) evaluated in exact rationals equals the integer form."""
    rng = random.Random(1)
    for _ in range(3000):
        total = rng.randint(1, 200000)
        fps = rng.choice([1.0, 10.0, 23.976, 24.0, 25.0, 29.97, 30.0, 59.94, 60.0, 7.5])
        tp = rng.choice([1, 2, 4])
        mx = rng.choice([tp, 16, 64, 128, 256, 768])
        n, idx = O.sample_frame_indices(total, fps, rng.choice([0.5, 1.0, 2.0, 4.0]), mx, tp)
        for i in range(0, n, max(1, n // 7)):
            assert idx[i] == min(total - 1, math.floor((Fraction(i) + Fraction(1, 2)) * total / n))


def test_sampling_invariants_bruteforce():
    """S:45-46 (sorted, unique, in range, <= max_frames), S:78 (multiple of tp when n >= tp),
    S:149 (monotone in max_frames) and C3 (n <= total)."""
    rng = random.Random(2)
    for _ in range(4000):
        total = rng.randint(1, 5000)
        fps = rng.uniform(0.5, 120.0)
        tfps = rng.choice([0.25, 1.0, 2.0, 3.0, 10.0])
        tp = rng.choice([1, 2, 3, 4])
        mx = rng.randint(tp, 300)
        n, idx = O.sample_frame_indices(total, fps, tfps, mx, tp)
        assert len(idx) == n and 1 <= n <= min(mx, total)
        assert all(0 <= a < total for a in idx)
        assert all(a < b for a, b in zip(idx, idx[1:]))
        if n >= tp:
            assert n % tp == 0
        else:
            assert n == total < tp
        n2, _ = O.sample_frame_indices(total, fps, tfps, mx + rng.randint(0, 50), tp)
        assert n2 >= n


def test_baseline_configs_frame_counts():
    """cfg1 n=8 (idx 0..7); cfg2 n=64; cfg3 n=768; 10 s of cfg2's source -> 20."""
    assert O.sample_frame_indices(8, 2.0, 2.0, 128, 2) == (8, list(range(8)))
    assert O.sample_frame_indices(1800, 30.0, 2.0, 64, 2)[0] == 64
    assert O.sample_frame_indices(300, 30.0, 2.0, 64, 2)[0] == 20
    assert O.sample_frame_indices(108000, 30.0, 2.0, 768, 2)[0] == 768


def test_effective_fps():
    assert O.effective_fps(20, 10.0, 100) == 2.0
    assert O.effective_fps(64, 30.0, 1800) == pytest.approx(64 / 60)


# ---------------- O2 smart_resize ----------------

def test_spec_smart_resize_examples(golden):
    for e in golden["smart_resize"]:
        assert O.smart_resize(e["h"], e["w"], e["budget"], e["factor"]) == tuple(e["out"]), e["cite"]


def test_paper_cache_size_reading(golden):
    """P:76 'roughly 360 MB' = 256 frames of a 720p clip resized at factor 28 under 262,144 px, 2 B/value."""
    e = golden["paper_cache_size"]
    H, W = O.smart_resize(e["h"], e["w"], e["budget"], e["factor"])
    assert (H, W) == (364, 672)
    mb = e["frames"] * H * W * 3 * e["bytes_per_value"] / 2**20
    assert abs(mb - e["approx_mb"]) / e["approx_mb"] < e["rel_tol"]


def test_round_half_even_div():
    assert O.round_half_even_div(720, 32) == 22      # 22.5 -> 22 (even), C5
    assert O.round_half_even_div(752, 32) == 24      # 23.5 -> 24
    for a in range(0, 2000):
        for f in (14, 16, 28, 32):
            assert O.round_half_even_div(a, f) == round(Fraction(a, f))   # Python's round = half-even


def test_smart_resize_matches_hf_library():
    """Library pin (C6): HF Qwen2-VL smart_resize (per-frame) and Qwen3-VL video smart_resize (total)."""
    from transformers.models.qwen2_vl.image_processing_qwen2_vl import smart_resize as hf2
    from transformers.models.qwen3_vl.video_processing_qwen3_vl import smart_resize as hf3
    rng = random.Random(3)
    for _ in range(20000):
        f = rng.choice([28, 32])
        h, w = rng.randint(f, 3000), rng.randint(f, 3000)
        if max(h, w) / min(h, w) > 200:
            continue
        b = rng.choice([f * f * 4, 100352, 262144, 1048576, rng.randint(f * f, 4_000_000)])
        mn = rng.choice([0, 3136, 16384])
        ref = hf2(h, w, factor=f, min_pixels=mn, max_pixels=b)
        if min(ref) >= f:          # HF can return 0 for tiny inputs; our reading floors at f
            assert O.smart_resize(h, w, b, f, mn) == ref, (h, w, b, f, mn)
        n = rng.randint(1, 800)
        tb = rng.choice([25165824, 12288 * 1024, 262144 * 64])
        ref3 = hf3(n, h, w, temporal_factor=2, factor=f, min_pixels=mn, max_pixels=tb)
        if min(ref3) >= f:
            assert O.smart_resize(h, w, tb, f, mn, n_frames=n, tp=2) == ref3


def test_smart_resize_closed_form_bounds_and_exact_crosscheck():
    """Bounds: multiples of f, >= f, area <= budget in the scaled branch; and the f64 answer is the
    exact-integer floor or one factor below it (rounding at exact-integer boundaries, C6)."""
    for f, b in [(28, 262144), (32, 262144), (32, 1048576), (28, 100352)]:
        for h in range(f, 3000, 37):
            for w in range(f, 3000, 41):
                H, W = O.smart_resize(h, w, b, f)
                assert H % f == 0 and W % f == 0 and H >= f and W >= f
                hb = max(f, f * O.round_half_even_div(h, f))
                wb = max(f, f * O.round_half_even_div(w, f))
                if hb * wb > b:
                    if H > f and W > f:
                        assert H * W <= b
                    eh, ew = O.smart_resize_exact_floor(h, w, b, f)
                    assert H in (eh, eh - f) and W in (ew, ew - f)
                else:
                    assert (H, W) == (hb, wb)


def test_baseline_config_resolutions():
    """SURVEY §8(a) H3."""
    assert O.smart_resize(128, 128, 262144, 32) == (128, 128)
    assert O.smart_resize(720, 1280, 262144, 32) == (384, 672)
    assert O.smart_resize(1080, 1920, 25165824, 32, n_frames=768, tp=2) == (128, 224)
    assert O.smart_resize(1080, 1920, 262144, 32) == (384, 672)
    assert O.smart_resize(1024, 1024, 1048576, 32) == (1024, 1024)
    assert O.smart_resize(720, 1280, 1048576, 32) == (704, 1280)   # half-to-even 22.5 -> 22 (C5)


# ---------------- O3 grid + whole plan ----------------

def test_spec_grid_examples(golden):
    for e in golden["compute_grid_thw"]:
        assert O.grid_thw(e["T"], e["H"], e["W"], e["patch"], e["tp"]) == tuple(e["grid"]), e["cite"]
    with pytest.raises(ValueError):
        O.grid_thw(2, 30, 28, 14, 2)


def test_spec_preprocess_example(golden):
    e = golden["preprocess_video"][0]
    pr = e["params"]
    params = I.qwen3_params(target_fps=pr["target_fps"], max_frames=pr["max_frames"],
                            video_max_pixels=pr["max_pixels"], patch_size=pr["patch"],
                            merge_size=pr["merge"], temporal_patch_size=pr["tp"])
    pl = O.plan_clip(params, I.clip(int(e["duration_s"] * e["source_fps"]), e["source_fps"], e["height"], e["width"]))
    assert pl.n == e["T"] and (pl.out_h, pl.out_w) == (e["out_h"], e["out_w"]) and pl.grid == tuple(e["grid"])


def test_spec_placeholder_counts(golden):
    for e in golden["validate_placeholder_alignment"]:
        t, h, w = e["grid"]
        assert t * h * w // e["merge"] ** 2 == e["features"]
        ids, _, st, _ = O.rope_index([np.full(e["placeholders"], 2)], [], [e["grid"]], e["merge"], variant=1)
        assert (st[0] == O.VP_OK) == e["ok"], e["cite"]


def test_plan_batch_offsets_cfg4():
    params, clips = I.config("cfg4")
    plans, tot = O.plan_batch(params, clips)
    assert tot["n_images"] == 16 and tot["n_videos"] == 8
    assert tot["img_tokens"] == 16 * 1024 and tot["vid_tokens"] == 8 * 8064
    assert tot["img_tokens"] + tot["vid_tokens"] == 80896
    assert [p.patch_offset for p in plans[:3]] == [0, 4096, 8192]
    assert [p.patch_offset for p in plans[16:19]] == [0, 32256, 64512]
    assert plans[17].group_offset == 32 and plans[17].grid_index == 1
    assert tot["indices"] == 16 + 8 * 64


def test_plan_invalid_clip_is_skipped():
    params = I.qwen3_params()
    plans, tot = O.plan_batch(params, [I.clip(0, 30.0, 64, 64), I.clip(10, 30.0, 64, 64), I.clip(5, 0.0, 64, 64)])
    assert [p.status for p in plans] == [O.VP_EINVAL, O.VP_OK, O.VP_EINVAL]
    assert tot["n_videos"] == 1 and plans[1].grid_index == 0


def test_dedup_keys_brute_force():
    """N3 oracle: first occurrence kept, batch order, every sample maps to a unique clip with its own key
    (brute force over all small key sequences)."""
    import itertools
    for n in range(0, 6):
        for keys in itertools.product(range(3), repeat=n):
            uid, ul = O.dedup_keys(list(keys))
            assert len(uid) == n and len(set(keys)) == len(ul)
            assert ul == sorted(ul) and all(keys[i] not in keys[:i] for i in ul)
            assert all(keys[ul[uid[k]]] == keys[k] and ul[uid[k]] <= k for k in range(n))
    uid, ul = O.dedup_keys([7] * 8 + [3] * 8)                      # GRPO: 2 prompts x 8 rollouts
    assert ul == [0, 8] and uid == [0] * 8 + [1] * 8


def test_hf_sampling_matches_hf_processor():
    """N1 oracle pin: sample_frame_indices_hf == HF Qwen3VLVideoProcessor.sample_frames (default fps 2, min 4,
    max 768) over random and edge metadata (total < 4, exact halves of linspace, long videos)."""
    import random
    from transformers.models.qwen3_vl.video_processing_qwen3_vl import Qwen3VLVideoProcessor
    from transformers.video_utils import VideoMetadata
    proc = Qwen3VLVideoProcessor()
    rng = random.Random(3)
    cases = [(1, 30.0), (2, 30.0), (3, 1.0), (7, 2.0), (100, 10.0), (1800, 30.0), (108000, 30.0), (13, 2.0),
             (61, 23.976)] + [(rng.randint(1, 50000), rng.choice([1.0, 24.0, 29.97, 30.0, 60.0, rng.uniform(0.3, 120)]))
                              for _ in range(400)]
    for total, fps in cases:
        ref = proc.sample_frames(VideoMetadata(total_num_frames=total, fps=fps))
        n, idx = O.sample_frame_indices_hf(total, fps, proc.fps, proc.min_frames, proc.max_frames)
        assert list(ref) == idx and n == len(ref), (total, fps)
