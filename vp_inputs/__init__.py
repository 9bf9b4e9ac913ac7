"""Seeded synthetic inputs shared by the oracle side and the CUDA side of the tests/bench.

This module holds NO arithmetic of the method (no sampling, resizing, normalising,
patchifying or position-id rule).  It only produces:

* u8 RGB frame content from counter-based formulas (identical on host and device:
  the device copy lives in ``vp_synth_frames`` and is checked bit-exactly against
  these functions by ``tests/test_inputs_gpu.py``);
* clip descriptors (source frame count, source fps, height, width, modality) that
  describe the BASELINE.json workloads;
* token-type sequences built from caller-supplied run lengths.

Frame content kinds
-------------------
``ramp``  : SPEC S:71 ``SyntheticVideoSpec``: (seed*2654435761 + i*97 + y*31 + x*7 + c) mod 256,
            with ``i`` the frame id passed in by the caller.
``noise`` : splitmix64 of the linear byte index ((i*H + y)*W + x)*3 + c plus the seed, top 8 bits.
            Uniform u8 -- the worst case for filter round-off.
"""
from __future__ import annotations

import numpy as np

KIND_RAMP = 0
KIND_NOISE = 1
_KINDS = {"ramp": KIND_RAMP, "noise": KIND_NOISE}

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def kind_id(kind: str | int) -> int:
    return _KINDS[kind] if isinstance(kind, str) else int(kind)


def _splitmix64(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def frames_u8(kind: str | int, seed: int, frame_ids, height: int, width: int) -> np.ndarray:
    """Return uint8 array (T, H, W, 3) for the given frame ids (THWC, RGB, row-major)."""
    k = kind_id(kind)
    fid = np.asarray(frame_ids, dtype=np.int64).reshape(-1, 1, 1, 1)
    y = np.arange(height, dtype=np.int64).reshape(1, -1, 1, 1)
    x = np.arange(width, dtype=np.int64).reshape(1, 1, -1, 1)
    c = np.arange(3, dtype=np.int64).reshape(1, 1, 1, 3)
    if k == KIND_RAMP:
        # the seed term is reduced mod 2^64 then mod 256 (only the low 8 bits matter).
        s = (int(seed) * 2654435761) % 256
        v = (s + fid * 97 + y * 31 + x * 7 + c) % 256
        return v.astype(np.uint8)
    if k == KIND_NOISE:
        lin = ((fid * height + y) * width + x) * 3 + c
        with np.errstate(over="ignore"):
            z = lin.astype(np.uint64) + np.uint64(int(seed) & 0xFFFFFFFFFFFFFFFF) * np.uint64(0xD1B54A32D192ED03)
        return (_splitmix64(z) >> np.uint64(56)).astype(np.uint8)
    raise ValueError(f"unknown kind {kind}")


# ---------------------------------------------------------------------------
# Workload descriptors (BASELINE.json configs).  Plain data, no method arithmetic.
# ---------------------------------------------------------------------------

def qwen3_params(**over) -> dict:
    """Qwen3-VL preset (patch 16, merge 2, temporal patch 2, mean/std 0.5) with the paper's
    training budgets (2 fps, 128 frames, 262,144 px/frame video, 1,048,576 px image)."""
    p = dict(target_fps=2.0, max_frames=128, temporal_patch_size=2, patch_size=16, merge_size=2,
             video_max_pixels=262144, image_max_pixels=1048576, min_pixels=0,
             budget_mode=0, sampling=0, mean=(0.5, 0.5, 0.5), std=(0.5, 0.5, 0.5), out_dtype=0)
    p.update(over)
    return p


def clip(total: int, fps: float, h: int, w: int, is_image: bool = False) -> dict:
    return dict(total_source_frames=int(total), source_fps=float(fps), height=int(h), width=int(w),
                is_image=bool(is_image))


def image(h: int, w: int) -> dict:
    return clip(1, 1.0, h, w, True)


def config(name: str):
    """Return (params, clips) for a BASELINE.json config name cfg1..cfg5."""
    if name == "cfg1":   # 8 u8 RGB frames 128x128 (source: 8 frames @ 2 fps)
        return qwen3_params(), [clip(8, 2.0, 128, 128)]
    if name == "cfg2":   # Qwen3-VL-8B RL clip: 30 fps 1280x720, 60 s, <=64 frames
        return qwen3_params(max_frames=64), [clip(1800, 30.0, 720, 1280)]
    if name == "cfg3":   # LVBench-shaped: 60 min 30 fps 1080p, 768 frames, total budget
        return (qwen3_params(max_frames=768, budget_mode=1, video_max_pixels=25165824),
                [clip(108000, 30.0, 1080, 1920)])
    if name == "cfg4":   # 16 images 1024^2 + 8 cfg2 videos
        return qwen3_params(max_frames=64), [image(1024, 1024)] * 16 + [clip(1800, 30.0, 720, 1280)] * 8
    if name == "cfg5":   # GRPO rollout batch: 512 cfg2 clips
        return qwen3_params(max_frames=64), [clip(1800, 30.0, 720, 1280)] * 512
    # other source resolutions at the cfg2 video budget, 16 clips of 60 s @ 30 fps each (bench side lines)
    res = {"res480p": (480, 854), "res1080p": (1080, 1920), "res1440p": (1440, 2560), "res2160p": (2160, 3840)}
    if name in res:
        h, w = res[name]
        return qwen3_params(max_frames=64), [clip(1800, 30.0, h, w)] * 16
    raise KeyError(name)


def token_types(runs) -> np.ndarray:
    """Build an int8 token-type sequence from [(type, length), ...]; 0 text, 1 image, 2 video."""
    out = [np.full(int(n), int(t), dtype=np.int8) for t, n in runs]
    return np.concatenate(out) if out else np.zeros(0, dtype=np.int8)
