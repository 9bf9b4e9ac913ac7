"""GPU checks of the C-ABI contract (include/vp.h "Conventions"): no device allocation and no state across calls,
reentrancy from several host threads on their own streams, the launch-mask hint, and the edges of the parameter
space the kernels must cover (odd patch size, negative std, downscales beyond the generic kernel's window tables:
the library is total over resize ratios)."""
import threading

import numpy as np
import pytest
import torch

import oracle as O
import vp_inputs as I
from parity import assert_pixels, host_frames, oracle_params, pack_frames

pytestmark = pytest.mark.gpu


def _batch():
    params, clips = I.config("cfg4")
    clips = clips[12:20] + [I.clip(9, 2.0, 70, 100), I.image(100, 60), I.image(2000, 3000)]
    return params, clips


def _setup(pre, clips):
    pl = pre.plan(clips)
    oplans, _ = O.plan_batch(oracle_params(pre.params), clips)
    fl = host_frames(oplans)
    buf, offs, pit = pack_frames(fl, [(3 * c["width"] + 15) // 16 * 16 for c in clips])
    return pl, oplans, fl, buf, offs, pit


def _run(pre, pl, buf, offs, pit, out, stream=None):
    import paper_2604_16893_b200 as vp
    vp.resize_normalize_patchify(pre.launch_params(pl), pl.plans_dev, pl.n, buf, offs, pit,
                                 out["pixel_values"] if out["pixel_values"].numel() else None,
                                 out["pixel_values_videos"], out["image_grid_thw"], out["video_grid_thw"],
                                 out["clip_status"], workspace=out["workspace"], stream=stream)


def test_no_device_memory_or_state_across_100_calls():
    """vp.h: the library never allocates device memory (scratch = the caller's workspace); 100 calls of the whole
    path on preallocated buffers leave the device's free memory unchanged."""
    import paper_2604_16893_b200 as vp
    params, clips = _batch()
    pre = vp.VisualPreprocessor(**params)
    pl, oplans, fl, buf, offs, pit = _setup(pre, clips)
    out = pre.alloc_outputs(pl)
    _run(pre, pl, buf, offs, pit, out)                   # first call: lazy module loading may map device memory
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(100):
        vp.plan_frames(pre.params, pl.clips_dev, pl.n, pl.plans_dev, pl.frame_indices, pl.totals_dev,
                       pl.group_timestamps)
        _run(pre, pl, buf, offs, pit, out)
    torch.cuda.synchronize()
    assert torch.cuda.mem_get_info()[0] == free0


def test_two_host_threads_two_streams_identical():
    """Reentrancy: two host threads, each on its own stream with its own outputs and workspace, 20 calls each,
    concurrently; every result is byte-identical to a serial run."""
    import paper_2604_16893_b200 as vp
    params, clips = _batch()
    pre = vp.VisualPreprocessor(**params)
    pl, oplans, fl, buf, offs, pit = _setup(pre, clips)
    ref = pre.alloc_outputs(pl)
    _run(pre, pl, buf, offs, pit, ref)
    torch.cuda.synchronize()
    outs = [pre.alloc_outputs(pl) for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    errors = []

    def work(t):
        try:
            with torch.cuda.stream(streams[t]):
                for _ in range(20):
                    _run(pre, pl, buf, offs, pit, outs[t], stream=streams[t])
            streams[t].synchronize()
        except Exception as e:                           # pragma: no cover - reported below
            errors.append(e)

    th = [threading.Thread(target=work, args=(t,)) for t in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors
    for o in outs:
        for k in ("pixel_values", "pixel_values_videos"):
            assert torch.equal(o[k].view(torch.int16), ref[k].view(torch.int16)), k


def test_launch_mask_hint_is_exact():
    """launch_mask = the plan's totals[VP_TOT_VARIANTS] skips absent variants only: identical bytes to mask 0
    (launch everything)."""
    import paper_2604_16893_b200 as vp
    params, clips = _batch()
    pre = vp.VisualPreprocessor(**params)
    pl, oplans, fl, buf, offs, pit = _setup(pre, clips)
    a, b = pre.alloc_outputs(pl), pre.alloc_outputs(pl)
    _run(pre, pl, buf, offs, pit, a)
    vp.resize_normalize_patchify(pre.params, pl.plans_dev, pl.n, buf, offs, pit, b["pixel_values"],
                                 b["pixel_values_videos"], b["image_grid_thw"], b["video_grid_thw"], b["clip_status"],
                                 workspace=b["workspace"])
    torch.cuda.synchronize()
    kv = set(pl.plans_host["kernel_variant"][: pl.n].tolist())
    assert int(pl.totals["variants"]) == sum(1 << v for v in kv)
    for k in ("pixel_values", "pixel_values_videos"):
        assert torch.equal(a[k].view(torch.int16), b[k].view(torch.int16)), k


def _parity(pre, clips, pitch_pad=0, align16=True):
    pl = pre.plan(clips)
    op = oracle_params(pre.params)
    oplans, _ = O.plan_batch(op, clips)
    fl = host_frames(oplans)
    pitches = [(3 * c["width"] + 15) // 16 * 16 if align16 else 3 * c["width"] + pitch_pad for c in clips]
    buf, offs, pit = pack_frames(fl, pitches)
    out = pre.run(pl, buf, offs, pit)
    torch.cuda.synchronize()
    ref = O.process_batch(op, clips, [f if f is not None else np.zeros((1, 1, 1, 3), np.uint8) for f in fl],
                          plans=oplans)
    assert out["clip_status"][: len(clips)].cpu().tolist() == [p.status for p in oplans]
    assert out["image_grid_thw"].cpu().tolist() == ref["image_grid_thw"].tolist()
    assert out["video_grid_thw"].cpu().tolist() == ref["video_grid_thw"].tolist()
    assert_pixels(out["pixel_values"].cpu(), ref["pixel_values_images"], "images")
    assert_pixels(out["pixel_values_videos"].cpu(), ref["pixel_values_videos"], "videos")
    return pl


KV_DIRECT = 7


@pytest.mark.parametrize("dtype", [1, 0])
def test_huge_downscales_take_the_direct_kernel(dtype):
    """Downscales beyond the generic kernel's 140-tap window tables (~34x per axis) are computed (KV_DIRECT, f64)
    rather than rejected: a 2000x3000 image and a 1500x2600 video at a 1024-pixel budget (-> 32x32, 47-94x), next
    to ordinary clips in the same call; temporal padding of the image into tp slots."""
    import paper_2604_16893_b200 as vp
    pre = vp.VisualPreprocessor(image_max_pixels=1024, video_max_pixels=1024, max_frames=3, out_dtype=dtype)
    clips = [I.image(2000, 3000), I.clip(5, 2.0, 1500, 2600), I.clip(9, 2.0, 70, 100), I.image(64, 64)]
    pl = _parity(pre, clips)
    kv = pl.plans_host["kernel_variant"][: len(clips)].tolist()
    assert kv[0] == KV_DIRECT and kv[1] == KV_DIRECT, kv


@pytest.mark.parametrize("align16", [True, False])
def test_odd_patch_size(align16):
    """ADVICE: odd patch sizes (p = 15, m = 1 and p = 7, m = 3) -- column pairs would straddle patches, so every
    clip takes the generic kernel; element-wise parity."""
    import paper_2604_16893_b200 as vp
    for p, m in ((15, 1), (7, 3)):
        f = p * m
        pre = vp.VisualPreprocessor(patch_size=p, merge_size=m, image_max_pixels=f * f * 60,
                                    video_max_pixels=f * f * 40, max_frames=3, out_dtype=1)
        clips = [I.image(200, 130), I.clip(5, 2.0, 90, 160), I.image(f * 4, f * 6)]
        pl = _parity(pre, clips, pitch_pad=1, align16=align16)
        assert 3 in pl.plans_host["kernel_variant"][: len(clips)].tolist()


@pytest.mark.parametrize("dtype", [1, 0])
def test_negative_std(dtype):
    """ADVICE: a negative std flips the order of the output-domain clamp bounds; parity on every kernel path
    (team, fast, copy, generic via an unaligned pitch)."""
    import paper_2604_16893_b200 as vp
    pre = vp.VisualPreprocessor(mean=(0.4, 0.5, 0.6), std=(-0.5, 0.25, -0.3), video_max_pixels=32768,
                                image_max_pixels=65536, max_frames=3, out_dtype=dtype)
    clips = [I.clip(7, 2.0, 250, 500), I.image(64, 96), I.image(150, 40), I.image(27, 27)]
    _parity(pre, clips)
    _parity(pre, clips, pitch_pad=3, align16=False)
