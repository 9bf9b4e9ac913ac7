"""Pins for oracle O4-O9 (AA bicubic weights, resize, normalise, pad, patchify, bf16 rounding).

* torch.nn.functional.interpolate(float64, bicubic, antialias=True) -- library pin of C10
* identity / constant-image special cases, partition of unity
* HF Qwen3VLVideoProcessor / Qwen2VLImageProcessor with do_resize=False -- library pin of C13-C17
* brute-force index loops for the patch permutation, and its inverse
* bf16 RNE by enumeration of neighbouring bf16 values (C15 / O9)
"""
import numpy as np
import pytest
import torch

import oracle as O
import vp_inputs as I


def _torch_aa(frame_u8, out_h, out_w):
    x = torch.from_numpy(frame_u8.astype(np.float64)).permute(2, 0, 1)[None]
    y = torch.nn.functional.interpolate(x, size=(out_h, out_w), mode="bicubic", antialias=True,
                                        align_corners=False)
    return y[0].permute(1, 2, 0).numpy()


@pytest.mark.parametrize("shape", [
    ((37, 53), (16, 32)),      # downscale, both axes
    ((96, 160), (64, 96)),     # mild downscale (cfg2-like ratio 1.5-1.7)
    ((270, 480), (32, 64)),    # strong downscale (cfg3-like ratio 8.4-7.5)
    ((20, 24), (32, 64)),      # upscale
    ((48, 64), (48, 32)),      # identity rows, downscale cols
    ((33, 31), (64, 16)),      # up rows, down cols
])
def test_resize_matches_torch_f64_antialias(shape):
    (h, w), (oh, ow) = shape
    fr = I.frames_u8("noise", 5, [0], h, w)[0]
    ours = O.resize_frame(fr, oh, ow)
    ref = np.clip(_torch_aa(fr, oh, ow), 0, 255)           # C12: clamp once after both passes
    assert np.max(np.abs(ours - ref)) < 1e-9


def test_identity_resize_is_exact_copy():
    fr = I.frames_u8("noise", 3, [0], 40, 56)[0]
    assert np.array_equal(O.resize_frame(fr, 40, 56), fr.astype(np.float64))
    for x0w in O.aa_weights(56, 56):
        x0, w = x0w
        assert set(np.unique(w)) <= {0.0, 1.0}


def test_weights_partition_of_unity_and_constant_image():
    for a, b in [(720, 384), (1280, 672), (1080, 128), (1920, 224), (17, 64), (5, 3)]:
        for x0, w in O.aa_weights(a, b):
            assert abs(w.sum() - 1.0) < 1e-12 and x0 >= 0 and x0 + len(w) <= a
    fr = np.full((45, 70, 3), 200, np.uint8)
    assert np.allclose(O.resize_frame(fr, 32, 64), 200.0, atol=1e-10)


def test_keys_kernel_closed_form():
    # Keys (a=-0.5): K(0)=1, K(+-1)=K(+-2)=0, K(0.5)=0.5625, K(1.5)=-0.0625, symmetric
    assert O.keys_cubic(0.0) == 1.0 and O.keys_cubic(1.0) == 0.0 and O.keys_cubic(2.0) == 0.0
    assert O.keys_cubic(0.5) == pytest.approx(0.5625) and O.keys_cubic(-1.5) == pytest.approx(-0.0625)


def test_resize_pixel_equals_full_frame():
    fr = I.frames_u8("noise", 9, [0], 91, 150)[0]
    full = O.resize_frame(fr, 48, 64)
    cache = {}
    rng = np.random.default_rng(0)
    for _ in range(200):
        i, j, c = rng.integers(48), rng.integers(64), rng.integers(3)
        assert abs(O.resize_pixel(fr, 48, 64, i, j, c, cache) - full[i, j, c]) < 1e-9


def test_patchify_bruteforce_index_formula():
    """O8 written as plain loops over (r, q) on a tiny odd-T input."""
    p, m, tp = 2, 2, 2
    T, H, W = 3, 8, 12
    x = np.arange(T * H * W * 3, dtype=np.float64).reshape(T, H, W, 3)
    got = O.patchify(x, p, m, tp)
    xp = np.concatenate([x, x[-1:]])                   # C16 repeat last frame
    gt, gh, gw = 2, H // p, W // p
    assert got.shape == (gt * gh * gw, 3 * tp * p * p)
    for t in range(gt):
        for hb in range(gh // m):
            for wb in range(gw // m):
                for mh in range(m):
                    for mw in range(m):
                        r = (((t * (gh // m) + hb) * (gw // m) + wb) * m + mh) * m + mw
                        for c in range(3):
                            for ti in range(tp):
                                for py in range(p):
                                    for px in range(p):
                                        q = ((c * tp + ti) * p + py) * p + px
                                        v = xp[t * tp + ti, (hb * m + mh) * p + py, (wb * m + mw) * p + px, c]
                                        assert got[r, q] == v
                                        assert O.patch_coords(r, q, (gt, gh, gw), p, m, tp) == (
                                            t * tp + ti, (hb * m + mh) * p + py, (wb * m + mw) * p + px, c)


def test_normalise_patchify_matches_hf_video_processor():
    """Library pin: HF Qwen3-VL video processor with do_resize=False on already-resized frames."""
    from transformers.models.qwen3_vl.video_processing_qwen3_vl import Qwen3VLVideoProcessor
    proc = Qwen3VLVideoProcessor()
    for T in (4, 5):                                    # even and odd T (temporal pad)
        fr = I.frames_u8("noise", T, list(range(T)), 64, 96)
        out = proc(videos=[torch.from_numpy(fr).permute(0, 3, 1, 2)], do_resize=False,
                   do_sample_frames=False, return_tensors="pt")
        ref = out["pixel_values_videos"].double().numpy()
        ours = O.patchify(O.normalize(fr.astype(np.float64), proc.image_mean, proc.image_std), 16, 2, 2)
        assert out["video_grid_thw"].tolist() == [[-(-T // 2), 4, 6]]
        assert np.max(np.abs(ours - ref)) < 1e-6      # HF computes in fp32


def test_normalise_patchify_matches_hf_image_processor():
    """Library pin: HF Qwen2-VL image processor (CLIP mean/std, patch 14): image -> tp copies."""
    from transformers.models.qwen2_vl.image_processing_qwen2_vl import Qwen2VLImageProcessor
    proc = Qwen2VLImageProcessor()
    fr = I.frames_u8("noise", 1, [0], 56, 84)
    out = proc(images=[torch.from_numpy(fr[0]).permute(2, 0, 1)], do_resize=False, return_tensors="pt")
    ref = out["pixel_values"].double().numpy()
    ours = O.patchify(O.normalize(fr.astype(np.float64), proc.image_mean, proc.image_std), 14, 2, 2)
    assert out["image_grid_thw"].tolist() == [[1, 4, 6]]
    assert np.max(np.abs(ours - ref)) < 2e-6


def test_bf16_rne_by_enumeration():
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.uniform(-1.1, 1.1, 20000), rng.normal(0, 1e-3, 2000), [0.0, 1.0, -1.0, 0.5]])
    bits = O.bf16_rne_bits(x)
    val = O.bf16_bits_to_f64(bits)
    for dv in (-1, 1):
        nb = (bits.astype(np.int64) + dv).astype(np.uint16)
        nv = O.bf16_bits_to_f64(nb)
        # nearest: no neighbour strictly closer; ties -> even mantissa
        ok = np.isfinite(nv) & (np.sign(nv) * np.sign(val) >= 0)   # same-sign finite neighbour
        d0, d1 = np.abs(x - val)[ok], np.abs(x - nv)[ok]
        assert np.all(d0 <= d1)
        assert np.all((bits[ok][d0 == d1] & 1) == 0)
    # exact ties constructed on purpose: halfway between 1.0 and 1.0078125
    assert O.bf16_bits_to_f64(O.bf16_rne_bits(np.array([1.0 + 2**-8])))[0] == 1.0
    assert O.bf16_bits_to_f64(O.bf16_rne_bits(np.array([1.0 + 3 * 2**-8])))[0] == 1.0 + 2**-6


def test_process_batch_end_to_end_small():
    params, clips = I.config("cfg1")
    plans, _ = O.plan_batch(params, clips)
    fr = I.frames_u8("ramp", 0, plans[0].idx, 128, 128)
    res = O.process_batch(params, clips, [fr])
    assert res["pixel_values_videos"].shape == (256, 1536)
    assert res["video_grid_thw"].tolist() == [[4, 8, 8]]
    # identity resize + mean/std 0.5: values are exactly v/127.5 - 1
    assert np.max(np.abs(res["pixel_values_videos"] - O.patchify(fr / 127.5 - 1.0, 16, 2, 2))) < 1e-12


def test_live_rows_bound():
    """The fast kernel's 5-slot vertical ring assumes <= 5 output rows are live at any source row when
    in/out > 0.8 (windows trimmed of exact-zero taps).  Brute force over many ratios."""
    import random
    rng = random.Random(0)
    cases = [(720, 384), (1080, 128), (1024, 1024), (999, 1000), (801, 1000), (27, 32), (1080, 1088)]
    for _ in range(1500):
        out = rng.randint(16, 900)
        inn = max(1, int(round(out * rng.uniform(0.801, 10.0))))
        cases.append((inn, out))
    for inn, out in cases:
        if inn / out <= 0.8:
            continue
        live = np.zeros(inn, dtype=int)
        for x0, w in O.aa_weights(inn, out):
            nz = np.nonzero(w)[0]
            live[x0 + nz[0]: x0 + nz[-1] + 1] += 1
        assert live.max() <= 5, (inn, out)


def test_column_pair_union_bound():
    """The fast kernel's horizontal pass loads the union of two adjacent output columns' (trimmed) windows:
    <= 11 / 23 / 51 pixels for the MILD / MEDIUM / STRONG tap classes (taps <= 9 / 18 / 40)."""
    import math
    import random
    rng = random.Random(1)
    limit = {0: 11, 1: 23, 2: 51}
    for _ in range(1500):
        out = rng.randint(16, 700)
        inn = max(1, int(round(out * rng.uniform(0.81, 9.5))))
        fs = max(inn / out, 1.0)
        taps = 1 if inn == out else math.floor(4 * fs) + 2
        var = 0 if taps <= 9 else (1 if taps <= 18 else 2)
        ws = []
        for x0, w in O.aa_weights(inn, out):
            nz = np.nonzero(w)[0]
            ws.append((x0 + nz[0], x0 + nz[-1] + 1))
        for j in range(0, len(ws) - 1, 2):
            assert ws[j + 1][1] - ws[j][0] <= limit[var], (inn, out, j)


def test_u8_resize_matches_torch_uint8_antialias():
    """N1 oracle pin: resize_frame_u8 == torch.nn.functional.interpolate(uint8, bicubic, antialias=True) bit for bit
    (the path HF's fast image / video processors take for uint8 frames), over down- and upscales, identity axes,
    ragged sizes and the cfg2 geometry (720p -> 384x672)."""
    import torch
    import torch.nn.functional as F
    rng = np.random.default_rng(11)
    shapes = [(720, 1280, 384, 672), (37, 53, 20, 30), (64, 96, 64, 40), (50, 50, 50, 30), (30, 40, 60, 80),
              (1, 7, 3, 2)] + [tuple(int(v) for v in rng.integers(1, 90, 4)) for _ in range(60)]
    for H, W, oh, ow in shapes:
        img = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
        ref = F.interpolate(torch.from_numpy(img).permute(2, 0, 1)[None], size=(oh, ow), mode="bicubic",
                            antialias=True)[0].permute(1, 2, 0).numpy()
        assert np.array_equal(O.resize_frame_u8(img, oh, ow), ref), (H, W, oh, ow)


def test_u8_resize_quantised_weights_sum():
    """Each quantised row of coefficients sums to 2^p within its rounding (|sum - 2^p| <= taps/2): the integer
    filter preserves a constant image up to rounding."""
    for inn, out in ((720, 384), (1280, 672), (30, 80), (7, 3)):
        q, p = O.quantize_weights_u8(inn, out)
        for _, c in q:
            assert abs(sum(c) - (1 << p)) <= len(c) / 2 + 1
        img = np.full((inn, 5, 3), 200, np.uint8)
        assert np.abs(O.resize_frame_u8(img, out, 5).astype(int) - 200).max() <= 1
