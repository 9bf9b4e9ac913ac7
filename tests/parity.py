"""Shared helpers for GPU-vs-oracle parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np
import torch

import oracle as O
import vp_inputs as I

F32_TOL = 1e-5          # north_star: |gpu - x| <= 1e-5 absolute in fp32
BF16_ABS = 1e-5         # C15 dual criterion: within RNE(x -+ 1e-5) ...
BF16_ULP = 1            # ... or within 1 bf16 ulp of RNE(x)


def oracle_params(vp_params) -> dict:
    p = vp_params
    return dict(target_fps=p.target_fps, max_frames=p.max_frames, temporal_patch_size=p.temporal_patch_size,
                patch_size=p.patch_size, merge_size=p.merge_size, video_max_pixels=p.video_max_pixels,
                image_max_pixels=p.image_max_pixels, min_pixels=p.min_pixels, budget_mode=p.budget_mode,
                sampling=p.sampling, mean=tuple(p.mean), std=tuple(p.std), out_dtype=p.out_dtype,
                min_frames=p.min_frames, resize_mode=p.resize_mode)


def _ord_bf16(bits: np.ndarray) -> np.ndarray:
    b = bits.astype(np.int64)
    return np.where(b & 0x8000, -(b & 0x7FFF), b)


def pixel_failures(gpu: torch.Tensor, ref: np.ndarray) -> np.ndarray:
    """Boolean mask of elements violating the parity bar (fp32: 1e-5 abs; bf16: C15)."""
    if gpu.dtype == torch.float32:
        return np.abs(gpu.numpy().astype(np.float64) - ref) > F32_TOL
    assert gpu.dtype == torch.bfloat16
    gbits = gpu.view(torch.int16).numpy().view(np.uint16)
    rbits = O.bf16_rne_bits(ref)
    ulp_ok = np.abs(_ord_bf16(gbits) - _ord_bf16(rbits)) <= BF16_ULP
    g = O.bf16_bits_to_f64(gbits)
    lo = O.bf16_bits_to_f64(O.bf16_rne_bits(ref - BF16_ABS))
    hi = O.bf16_bits_to_f64(O.bf16_rne_bits(ref + BF16_ABS))
    return ~(ulp_ok | ((g >= lo) & (g <= hi)))


def assert_pixels(gpu: torch.Tensor, ref: np.ndarray, what: str = ""):
    assert tuple(gpu.shape) == tuple(ref.shape), (what, gpu.shape, ref.shape)
    bad = pixel_failures(gpu, ref)
    if bad.any():
        i = np.argwhere(bad)[0]
        gv = gpu.float().numpy()[tuple(i)]
        raise AssertionError(f"{what}: {int(bad.sum())} of {bad.size} pixels outside tolerance; first at {i.tolist()}:"
                             f" gpu {gv!r} oracle {ref[tuple(i)]!r}")


def host_frames(plans_oracle, kind="noise", seed_base=0):
    """Per clip, the u8 sampled frames the GPU side will also see (content id = source index)."""
    out = []
    for k, pl in enumerate(plans_oracle):
        if pl.status != O.VP_OK:
            out.append(None)
            continue
        out.append(I.frames_u8(kind, seed_base + k, pl.idx, pl.in_h, pl.in_w))
    return out


def pack_frames(frames_list, pitches, device="cuda"):
    """Pack host frames into one device buffer with the given per-clip row pitches."""
    offs, cur = [], 0
    for fr, pitch in zip(frames_list, pitches):
        offs.append(cur)
        if fr is not None:
            cur += fr.shape[0] * fr.shape[1] * pitch
    buf = np.zeros(max(cur, 16), dtype=np.uint8)
    for fr, pitch, off in zip(frames_list, pitches, offs):
        if fr is None:
            continue
        T, H, W, _ = fr.shape
        view = buf[off: off + T * H * pitch].reshape(T, H, pitch)
        view[:, :, : 3 * W] = fr.reshape(T, H, 3 * W)
    return (torch.from_numpy(buf).to(device), torch.tensor(offs, dtype=torch.int64, device=device),
            torch.tensor(pitches, dtype=torch.int64, device=device))
