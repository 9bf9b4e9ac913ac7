"""N4 on the GPU, bit-exact vs the oracle: vp_nv12_to_rgb (decoder NV12 surfaces with padded pitch and frame stride,
written straight into a K3 frame-buffer slot, then resized by K3) and vp_vision_ids (vision-tower patch ids and
cu_seqlens from the grids K3 emits)."""
import numpy as np
import pytest
import torch

import oracle as O
import vp_inputs as I
from parity import assert_pixels, oracle_params

pytestmark = pytest.mark.gpu


def _nv12_frames(rng, n, H, W, pitch, stride):
    buf = np.zeros(n * stride, np.uint8)
    planes = []
    for f in range(n):
        y = rng.integers(0, 256, (H, W), dtype=np.uint8)
        uv = rng.integers(0, 256, (H // 2, W), dtype=np.uint8)
        base = f * stride
        for r in range(H):
            buf[base + r * pitch: base + r * pitch + W] = y[r]
        for r in range(H // 2):
            buf[base + (H + r) * pitch: base + (H + r) * pitch + W] = uv[r]
        planes.append((y, uv))
    return buf, planes


@pytest.mark.parametrize("H,W", [(2, 2), (24, 40), (50, 86)])
def test_nv12_to_rgb_bit_exact(H, W):
    import paper_2604_16893_b200 as vp
    rng = np.random.default_rng(H * W)
    n, pitch = 3, W + 64                              # NVDEC-like padded pitch; UV plane right after the Y plane
    stride = pitch * (H + H // 2) + 128
    buf, planes = _nv12_frames(rng, n, H, W, pitch, stride)
    d = torch.from_numpy(buf).cuda()
    rgb_pitch = (3 * W + 15) // 16 * 16
    out = torch.full((n * H * rgb_pitch,), 7, dtype=torch.uint8, device="cuda")
    vp.nv12_to_rgb(d, d[H * pitch:], pitch, stride, H, W, n, out, rgb_pitch, H * rgb_pitch)
    got = out.cpu().numpy().reshape(n, H, rgb_pitch)
    for f, (y, uv) in enumerate(planes):
        assert np.array_equal(got[f, :, : 3 * W].reshape(H, W, 3), O.nv12_to_rgb(y, uv)), f
        assert (got[f, :, 3 * W:] == 7).all()            # padding untouched


def test_nv12_into_k3_end_to_end():
    """decoder NV12 -> vp_nv12_to_rgb into the clip's frame slot -> K3 (team kernel) vs the oracle on the oracle's RGB."""
    import paper_2604_16893_b200 as vp
    rng = np.random.default_rng(5)
    pre = vp.VisualPreprocessor(max_frames=4, video_max_pixels=16384, out_dtype=1)
    clip = I.clip(4, 2.0, 96, 160)
    pl = pre.plan([clip])
    n = int(pl.plans_host["n_frames"][0])
    H, W, pitch = 96, 160, 256
    stride = pitch * (H + H // 2)
    buf, planes = _nv12_frames(rng, n, H, W, pitch, stride)
    d = torch.from_numpy(buf).cuda()
    off, rp, total = pre.frames_layout(pl)
    frames = torch.zeros(total, dtype=torch.uint8, device="cuda")
    vp.nv12_to_rgb(d, d[H * pitch:], pitch, stride, H, W, n, frames[int(off[0]):], int(rp[0]), H * int(rp[0]))
    out = pre.run(pl, frames, torch.from_numpy(off).cuda(), torch.from_numpy(rp).cuda())
    rgb = np.stack([O.nv12_to_rgb(y, uv) for y, uv in planes])
    op = oracle_params(pre.params)
    ref = O.process_batch(op, [clip], [rgb])
    assert_pixels(out["pixel_values_videos"].cpu(), ref["pixel_values_videos"], "nv12 -> K3")


def test_vision_ids_bit_exact():
    import paper_2604_16893_b200 as vp
    grids = [(32, 24, 42), (1, 64, 64), (3, 16, 32), (1, 2, 2), (768, 8, 14)]
    pos, cu = vp.vision_ids(torch.tensor(grids, dtype=torch.int64, device="cuda"), 2)
    assert np.array_equal(pos.cpu().numpy().astype(np.int64), O.vision_pos_ids(grids, 2))
    assert cu.cpu().tolist() == O.vision_cu_seqlens(grids)
    pos, cu = vp.vision_ids(torch.zeros((0, 3), dtype=torch.int64, device="cuda"), 2)
    assert pos.numel() == 0 and cu.cpu().tolist() == [0]
