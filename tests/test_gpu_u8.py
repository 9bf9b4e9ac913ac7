"""N1 pixels on the GPU: VP_RESIZE_U8 (HF drop-in: torch's uint8 antialiased bicubic, pinned bit-exact to torch in
tests/test_oracle_pixels.py) -- the integer intermediate recovered from the f32 output equals the oracle's
resize_frame_u8 exactly, and the normalised pixels are within the C15 / 1e-5 bars; downscales past 15.5x report
VP_EUNSUPPORTED."""
import numpy as np
import pytest
import torch

import oracle as O
import vp_inputs as I
from parity import assert_pixels, host_frames, oracle_params, pack_frames

pytestmark = pytest.mark.gpu


def _run(pre, clips):
    pl = pre.plan(clips)
    op = oracle_params(pre.params)
    oplans, _ = O.plan_batch(op, clips)
    fl = host_frames(oplans)
    buf, offs, pit = pack_frames(fl, [(3 * c["width"] + 15) // 16 * 16 for c in clips])
    out = pre.run(pl, buf, offs, pit, strict=False)
    torch.cuda.synchronize()
    return pl, op, oplans, fl, out


@pytest.mark.parametrize("dtype", [1, 0])
def test_u8_mode_matches_oracle(dtype):
    import paper_2604_16893_b200 as vp
    pre = vp.VisualPreprocessor(max_frames=5, video_max_pixels=40000, image_max_pixels=65536, out_dtype=dtype,
                                resize_mode=vp.VP_RESIZE_U8, sampling=vp.VP_SAMPLE_LINSPACE, mean=(0.48, 0.45, 0.40),
                                std=(0.26, 0.26, 0.27))
    clips = [I.clip(40, 10.0, 250, 500), I.image(300, 200), I.clip(9, 2.0, 70, 100), I.image(64, 96),
             I.clip(3, 1.0, 20, 30), I.clip(12, 4.0, 720, 1280), I.image(33, 257)]
    pl, op, oplans, fl, out = _run(pre, clips)
    assert set(pl.plans_host["kernel_variant"][: len(clips)].tolist()) == {9}
    assert out["clip_status"][: len(clips)].cpu().tolist() == [0] * len(clips)
    ref = O.process_batch(op, clips, fl, plans=oplans)
    assert_pixels(out["pixel_values"].cpu(), ref["pixel_values_images"], "images")
    assert_pixels(out["pixel_values_videos"].cpu(), ref["pixel_values_videos"], "videos")
    if dtype == 1:
        # the integer intermediate, recovered from x = v*scale_c + bias_c, is the oracle's (torch's) bit for bit
        p, m, tp = op["patch_size"], op["merge_size"], op["temporal_patch_size"]
        pv = out["pixel_values_videos"].cpu().numpy()
        o = oplans[5]
        row0 = sum(q.patches for q in oplans[:5] if not q.is_image)
        scale = np.array([1.0 / (255.0 * s) for s in op["std"]])
        bias = np.array([-mu / s for mu, s in zip(op["mean"], op["std"])])
        for f in range(o.n):
            want = O.resize_frame_u8(fl[5][f], o.out_h, o.out_w)
            for y, x in ((0, 0), (o.out_h - 1, o.out_w - 1), (o.out_h // 2, 37), (100, o.out_w - 3)):
                for c in range(3):
                    r, q = None, None
                    hb, mh, py = y // (p * m), (y // p) % m, y % p
                    wb, mw, px = x // (p * m), (x // p) % m, x % p
                    g, ti = f // tp, f % tp
                    r = row0 + (((g * (o.grid[1] // m) + hb) * (o.grid[2] // m) + wb) * m + mh) * m + mw
                    q = ((c * tp + ti) * p + py) * p + px
                    v = (pv[r, q] - bias[c]) / scale[c]
                    assert abs(v - round(v)) < 1e-3 and int(round(v)) == int(want[y, x, c]), (f, y, x, c)


def test_u8_mode_unsupported_ratio():
    import paper_2604_16893_b200 as vp
    pre = vp.VisualPreprocessor(image_max_pixels=1024, resize_mode=vp.VP_RESIZE_U8)
    clips = [I.image(2000, 3000), I.image(64, 64)]
    pl, op, oplans, fl, out = _run(pre, clips)
    assert out["clip_status"][:2].cpu().tolist() == [vp.VP_EUNSUPPORTED, 0]
    with pytest.raises(vp.VpError):
        pre.run(pl, *pack_frames(fl, [(3 * c["width"] + 15) // 16 * 16 for c in clips]))


def test_u8_mode_any_alignment():
    """The u8 kernel reads bytes: clips with unaligned pitches, and a frame buffer whose base is not 16-B aligned,
    still take it (not the float generic kernel)."""
    import paper_2604_16893_b200 as vp
    pre = vp.VisualPreprocessor(max_frames=3, video_max_pixels=20000, image_max_pixels=30000, out_dtype=1,
                                resize_mode=vp.VP_RESIZE_U8)
    clips = [I.clip(7, 2.0, 70, 100), I.image(90, 61), I.image(33, 257)]
    pl = pre.plan(clips)
    op = oracle_params(pre.params)
    oplans, _ = O.plan_batch(op, clips)
    fl = host_frames(oplans)
    buf, offs, pit = pack_frames(fl, [3 * c["width"] + 1 for c in clips])           # unaligned pitches
    shifted = torch.zeros(buf.numel() + 3, dtype=torch.uint8, device="cuda")
    shifted[3:] = buf                                                                  # base off by 3 bytes
    out = pre.run(pl, shifted[3:], offs, pit)
    torch.cuda.synchronize()
    ref = O.process_batch(op, clips, fl, plans=oplans)
    assert_pixels(out["pixel_values"].cpu(), ref["pixel_values_images"], "images")
    assert_pixels(out["pixel_values_videos"].cpu(), ref["pixel_values_videos"], "videos")
