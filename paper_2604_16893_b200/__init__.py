"""B200-native visual-preprocessing hot path of EasyVideoR1 (arXiv 2604.16893).

Thin Python binding over the C ABI in ``include/vp.h`` (libvp.so, hand-written sm_100a CUDA).
Every step of the path runs in the library's kernels; this module only marshals torch tensors
(device memory, streams) into the ABI and, for the convenience API, sizes outputs and raises on
device-reported errors (strict by default).  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from .presets import PRESETS, preset
from ._lib import (DESC_DTYPE, PLAN_DTYPE, TOT, TOT_LEN, VP_BUDGET_PER_FRAME, VP_BUDGET_TOTAL, VP_ECAPACITY,
                   VP_EINVAL, VP_EMISMATCH, VP_EUNSUPPORTED, VP_OK, VP_OUT_BF16, VP_OUT_F32, VP_ROPE_QWEN2,
                   VP_ROPE_QWEN3_SPLIT, VP_ROPE_QWEN25, VP_RESIZE_FLOAT, VP_RESIZE_U8, VP_SAMPLE_CENTER_BIN,
                   VP_SAMPLE_LINSPACE, VP_SYNTH_NOISE,
                   VP_SYNTH_RAMP, VpError, VpParams,
                   check, lib)

__all__ = [
    "make_params", "clip_desc_array", "plan_frames", "resize_normalize_patchify", "resize_workspace_bytes",
    "resize_workspace", "rope_index",
    "rope_index_workspace_bytes", "plan_records", "pack_offsets", "synth_frames", "dedup_clips", "dedup_views",
    "plan_second_per_grid", "preset", "PRESETS", "nv12_to_rgb", "vision_ids",
    "VisualPreprocessor",
    "PlacementMismatch", "VpError", "VpParams", "DESC_DTYPE", "PLAN_DTYPE", "TOT", "TOT_LEN",
    "VP_ROPE_QWEN3_SPLIT", "VP_ROPE_QWEN2", "VP_ROPE_QWEN25", "VP_OUT_BF16", "VP_OUT_F32",
    "VP_SAMPLE_CENTER_BIN", "VP_SAMPLE_LINSPACE", "VP_RESIZE_FLOAT", "VP_RESIZE_U8",
    "VP_BUDGET_PER_FRAME", "VP_BUDGET_TOTAL", "VP_SYNTH_RAMP", "VP_SYNTH_NOISE", "VP_OK", "VP_EINVAL",
    "VP_EMISMATCH", "VP_ECAPACITY", "VP_EUNSUPPORTED", "lib",
]


class PlacementMismatch(RuntimeError):
    """Strict-failure policy: placeholder tokens != visual features."""


# ---------------------------------------------------------------------------------------------
# marshalling helpers
# ---------------------------------------------------------------------------------------------

def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def make_params(target_fps=2.0, max_frames=128, temporal_patch_size=2, patch_size=16, merge_size=2,
                video_max_pixels=262144, image_max_pixels=1048576, min_pixels=0, budget_mode=0, sampling=0,
                mean=(0.5, 0.5, 0.5), std=(0.5, 0.5, 0.5), out_dtype=VP_OUT_BF16, min_frames=None, resize_mode=0) -> VpParams:
    """vp_params (defaults = Qwen3-VL preset with the P:271 budgets)."""
    p = VpParams()
    p.target_fps, p.max_frames, p.temporal_patch_size = float(target_fps), int(max_frames), int(temporal_patch_size)
    p.patch_size, p.merge_size = int(patch_size), int(merge_size)
    p.video_max_pixels, p.image_max_pixels, p.min_pixels = int(video_max_pixels), int(image_max_pixels), int(min_pixels)
    p.budget_mode, p.sampling, p.out_dtype = int(budget_mode), int(sampling), int(out_dtype)
    p.min_frames = min(4, p.max_frames) if min_frames is None else int(min_frames)   # HF Qwen3-VL: 4
    p.resize_mode = int(resize_mode)
    for c in range(3):
        p.mean[c], p.std[c] = float(mean[c]), float(std[c])
    return p


def clip_desc_array(clips) -> np.ndarray:
    """list of dicts (total_source_frames, source_fps, height, width, is_image) -> vp_clip_desc[]."""
    a = np.zeros(len(clips), dtype=DESC_DTYPE)
    for k, c in enumerate(clips):
        a[k] = (int(c["total_source_frames"]), float(c["source_fps"]), int(c["height"]), int(c["width"]),
                int(bool(c.get("is_image", False))), 0)
    return a


def plan_frames(params: VpParams, clips, n: int, plans, frame_indices, totals, group_timestamps=None,
                stream=None) -> None:
    """vp_plan_frames.  clips/plans: uint8 device tensors holding vp_clip_desc[n] / vp_clip_plan[n]."""
    check(lib.vp_plan_frames(C.byref(params), _ptr(clips), int(n), _ptr(plans), _ptr(frame_indices),
                             frame_indices.numel() if frame_indices is not None else 0, _ptr(group_timestamps),
                             group_timestamps.numel() if group_timestamps is not None else 0, _ptr(totals),
                             _stream(stream)), "vp_plan_frames")


def resize_workspace_bytes(n: int) -> int:
    return int(lib.vp_resize_workspace_bytes(int(n)))


def resize_workspace(n: int, device) -> torch.Tensor:
    """Caller-owned scratch for vp_resize_normalize_patchify (256-B aligned by the torch allocator)."""
    return torch.empty(max(resize_workspace_bytes(n), 256), dtype=torch.uint8, device=device)


def resize_normalize_patchify(params: VpParams, plans, n: int, frames, clip_byte_offset, row_pitch,
                              pixel_values_images, pixel_values_videos, image_grid_thw, video_grid_thw,
                              clip_status=None, workspace=None, stream=None, first_clip: int = 0) -> None:
    """vp_resize_normalize_patchify (O4-O9) for clips [first_clip, first_clip+n) of a plan array.
    ``workspace``: uint8 device tensor of >= resize_workspace_bytes(n) bytes (allocated here if None)."""
    D = 3 * params.temporal_patch_size * params.patch_size ** 2
    icap = pixel_values_images.numel() // D if pixel_values_images is not None else 0
    vcap = pixel_values_videos.numel() // D if pixel_values_videos is not None else 0
    k0 = int(first_clip)
    pp = plans.data_ptr() + k0 * PLAN_DTYPE.itemsize
    co = clip_byte_offset.data_ptr() + 8 * k0
    rp = row_pitch.data_ptr() + 8 * k0
    cs = clip_status.data_ptr() + 4 * k0 if clip_status is not None else None
    if workspace is None:
        workspace = resize_workspace(n, frames.device)
    check(lib.vp_resize_normalize_patchify(C.byref(params), pp, int(n), _ptr(frames), co, rp,
                                           _ptr(pixel_values_images),
                                           icap, _ptr(pixel_values_videos), vcap, _ptr(image_grid_thw),
                                           _ptr(video_grid_thw), cs, _ptr(workspace), workspace.numel(),
                                           _stream(stream)),
          "vp_resize_normalize_patchify")


def rope_index_workspace_bytes(B: int, n_videos: int) -> int:
    return int(lib.vp_rope_index_workspace_bytes(int(B), int(n_videos)))


def rope_index(params: VpParams, variant: int, mm_token_type, cu_seqlens, image_grid_thw, video_grid_thw,
               position_ids, rope_deltas, seq_status, workspace, second_per_grid=None, tokens_per_second=0,
               stream=None) -> None:
    """vp_rope_index (O11).  position_ids: int64 [3, total_L]; seq_status: int32 [B+1]."""
    B = cu_seqlens.numel() - 1
    ni = image_grid_thw.shape[0] if image_grid_thw is not None else 0
    nv = video_grid_thw.shape[0] if video_grid_thw is not None else 0
    check(lib.vp_rope_index(C.byref(params), int(variant), _ptr(mm_token_type), _ptr(cu_seqlens), int(B),
                            int(mm_token_type.numel()), _ptr(image_grid_thw), int(ni), _ptr(video_grid_thw),
                            int(nv), _ptr(second_per_grid), int(tokens_per_second), _ptr(position_ids),
                            _ptr(rope_deltas), _ptr(seq_status), _ptr(workspace), workspace.numel(),
                            _stream(stream)), "vp_rope_index")


def plan_records(plans, n: int, merge_size: int, records, stream=None) -> None:
    check(lib.vp_plan_records(_ptr(plans), int(n), int(merge_size), _ptr(records), _stream(stream)),
          "vp_plan_records")


def pack_offsets(gathered, world: int, clips_per_rank: int, token_offsets, patch_offsets, stream=None) -> None:
    check(lib.vp_pack_offsets(_ptr(gathered), int(world), int(clips_per_rank), _ptr(token_offsets),
                              _ptr(patch_offsets), _stream(stream)), "vp_pack_offsets")


def synth_frames(kind: int, seed: int, frame_ids, height: int, width: int, out, row_pitch=None, stream=None) -> None:
    """vp_synth_frames: test/bench input generator (S:71 ramp or splitmix noise), never timed."""
    pitch = 3 * width if row_pitch is None else int(row_pitch)
    check(lib.vp_synth_frames(int(kind), int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(frame_ids), int(frame_ids.numel()),
                              int(height), int(width), pitch, _ptr(out), _stream(stream)), "vp_synth_frames")


def plan_second_per_grid(clips, plans, n: int, temporal_patch_size: int, second_per_grid, stream=None) -> None:
    """vp_plan_second_per_grid (N2, Qwen2.5-VL): f64 [n_videos] seconds per temporal grid."""
    check(lib.vp_plan_second_per_grid(_ptr(clips), _ptr(plans), int(n), int(temporal_patch_size),
                                      _ptr(second_per_grid), _stream(stream)), "vp_plan_second_per_grid")


def nv12_to_rgb(y, uv, pitch: int, frame_stride: int, height: int, width: int, n_frames: int, rgb, rgb_pitch: int,
                rgb_frame_stride: int, stream=None) -> None:
    """vp_nv12_to_rgb (N4): NVDEC NV12 planes -> u8 RGB THWC frames (BT.601 limited, OpenCV fixed point).
    y / uv / rgb may be uint8 tensors or (tensor, byte offset) views; pointers are taken from them as given."""
    check(lib.vp_nv12_to_rgb(_ptr(y), _ptr(uv), int(pitch), int(frame_stride), int(height), int(width),
                             int(n_frames), _ptr(rgb), int(rgb_pitch), int(rgb_frame_stride), _stream(stream)),
          "vp_nv12_to_rgb")


def vision_ids(grid_thw, merge_size: int, stream=None):
    """vp_vision_ids (N4): per pixel_values row its (row, col) patch ids [P,2] int32 and cu_seqlens [sum t + 1]."""
    g = grid_thw.contiguous()
    n = g.shape[0]
    gl = g.cpu().tolist()
    P = sum(t * h * w for t, h, w in gl)
    T = sum(t for t, _, _ in gl)
    pos = torch.empty(max(P, 1), 2, dtype=torch.int32, device=g.device)
    cu = torch.empty(T + 1, dtype=torch.int32, device=g.device)
    ws = torch.empty(int(lib.vp_vision_ids_workspace_bytes(n)), dtype=torch.uint8, device=g.device)
    check(lib.vp_vision_ids(_ptr(g), int(n), int(merge_size), _ptr(pos), _ptr(cu), _ptr(ws), ws.numel(),
                            _stream(stream)), "vp_vision_ids")
    return pos[:P], cu


def dedup_clips(keys, unique_id, unique_list, n_unique, stream=None) -> None:
    """vp_dedup_clips (N3).  keys: uint64 (or int64) device tensor [n]; outputs int32 [n], [n], [1]."""
    check(lib.vp_dedup_clips(_ptr(keys), int(keys.numel()), _ptr(unique_id), _ptr(unique_list), _ptr(n_unique),
                             _stream(stream)), "vp_dedup_clips")


def dedup_views(unique_plans, unique_id, patch_offset, grid_thw, status=None, stream=None) -> None:
    """vp_dedup_views (N3): per sample, its patch offset and grid in the unique clips' outputs."""
    check(lib.vp_dedup_views(_ptr(unique_plans), _ptr(unique_id), int(unique_id.numel()), _ptr(patch_offset),
                             _ptr(grid_thw), _ptr(status), _stream(stream)), "vp_dedup_views")


# ---------------------------------------------------------------------------------------------
# Convenience API: the whole path for a batch of clips (what a trainer calls)
# ---------------------------------------------------------------------------------------------

@dataclass
class Plan:
    n: int
    clips_dev: torch.Tensor
    plans_dev: torch.Tensor
    frame_indices: torch.Tensor
    group_timestamps: torch.Tensor
    totals_dev: torch.Tensor
    totals: dict | None = None
    plans_host: np.ndarray | None = None


class VisualPreprocessor:
    """plan -> (frames) -> pixel_values/grid_thw -> MRoPE ids, all on one CUDA device.

    Frames for clip k are its n_k sampled frames (u8 THWC); ``frames_layout(plan)`` gives the byte
    offsets of a packed frame buffer, so a decoder can write them directly (codec is out of scope).
    """

    def __init__(self, device="cuda", **params):
        self.device = torch.device(device)
        self.rope_variant = params.pop("rope_variant", VP_ROPE_QWEN3_SPLIT)
        self.tokens_per_second = params.pop("tokens_per_second", 0)
        self.params = make_params(**params)
        self.D = 3 * self.params.temporal_patch_size * self.params.patch_size ** 2

    # -- H1-H4, H9 --
    def plan(self, clips, stream=None, sync=True) -> Plan:
        n = len(clips)
        desc = torch.from_numpy(clip_desc_array(clips).view(np.uint8)).to(self.device)
        plans = torch.empty(max(n, 1) * PLAN_DTYPE.itemsize, dtype=torch.uint8, device=self.device)
        cap_idx = sum(1 if c.get("is_image") else self.params.max_frames for c in clips)
        cap_ts = sum(0 if c.get("is_image") else -(-self.params.max_frames // self.params.temporal_patch_size)
                     for c in clips)
        idx = torch.empty(max(cap_idx, 1), dtype=torch.int64, device=self.device)
        ts = torch.empty(max(cap_ts, 1), dtype=torch.float64, device=self.device)
        tot = torch.empty(TOT_LEN, dtype=torch.int64, device=self.device)
        plan_frames(self.params, desc, n, plans, idx, tot, ts, stream=stream)
        pl = Plan(n, desc, plans, idx, ts, tot)
        if sync:
            self.fetch(pl)
        return pl

    def fetch(self, pl: Plan) -> Plan:
        t = pl.totals_dev.cpu().tolist()
        pl.totals = {k: t[v] for k, v in TOT.items()}
        pl.plans_host = pl.plans_dev.cpu().numpy()[: pl.n * PLAN_DTYPE.itemsize].view(PLAN_DTYPE).copy()
        return pl

    def frames_layout(self, pl: Plan, row_align: int = 16):
        """Packed layout of every valid clip's sampled frames: (clip_byte_offset, row_pitch, total bytes).
        Rows are padded to 16 B by default so every clip can take the TMA kernels (unaligned rows fall back to
        the generic kernel)."""
        ph = pl.plans_host
        off = np.zeros(pl.n, dtype=np.int64)
        pitch = np.zeros(pl.n, dtype=np.int64)
        cur = 0
        for k in range(pl.n):
            pitch[k] = -(-3 * int(ph["in_w"][k]) // row_align) * row_align
            off[k] = cur
            if ph["status"][k] == VP_OK:
                cur += int(ph["n_frames"][k]) * int(ph["in_h"][k]) * int(pitch[k])
        return off, pitch, cur

    def launch_params(self, pl: Plan) -> VpParams:
        """self.params with the plan's kernel-variant mask as the launch hint (vp_params.launch_mask)."""
        p = VpParams()
        C.pointer(p)[0] = self.params
        p.launch_mask = int(pl.totals["variants"]) if pl.totals is not None else 0
        return p

    @classmethod
    def from_preset(cls, name: str, device="cuda", **overrides):
        """N2: a preprocessor for a model family (Qwen2-VL, Qwen2.5-VL, Qwen3-VL, Qwen3.5; see presets.py)."""
        p, rope = preset(name, **overrides)
        return cls(device=device, **p, **rope)

    def second_per_grid(self, pl: Plan, stream=None) -> torch.Tensor:
        """Per video of the plan (grid order), temporal_patch_size / HF sampled fps (Qwen2.5-VL time scale)."""
        nv = int(pl.totals["n_videos"]) if pl.totals is not None else pl.n
        out = torch.zeros(max(nv, 1), dtype=torch.float64, device=self.device)
        plan_second_per_grid(pl.clips_dev, pl.plans_dev, pl.n, self.params.temporal_patch_size, out, stream=stream)
        return out[:nv]

    def dedup(self, clips, keys, stream=None):
        """N3: keep the first occurrence of each key.  Returns (unique clips (list), unique_list (host int list),
        unique_id (device int32 [n]))."""
        n = len(clips)
        k = torch.as_tensor(np.asarray(keys, dtype=np.int64), device=self.device)
        uid = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        ul = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        nu = torch.empty(1, dtype=torch.int32, device=self.device)
        dedup_clips(k[:n], uid[:n], ul, nu, stream=stream)
        u = int(nu.item())
        ulist = ul[:u].cpu().tolist()
        return [clips[i] for i in ulist], ulist, uid[:n]

    def views(self, unique_plan: Plan, unique_id, stream=None):
        """N3: per-sample (patch_offset into the unique pixel_values, grid_thw, status) on the device."""
        n = unique_id.numel()
        po = torch.empty(max(n, 1), dtype=torch.int64, device=self.device)
        g = torch.empty(max(n, 1), 3, dtype=torch.int64, device=self.device)
        st = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        dedup_views(unique_plan.plans_dev, unique_id, po[:n], g[:n], st[:n], stream=stream)
        return po[:n], g[:n], st[:n]

    def alloc_outputs(self, pl: Plan):
        dt = torch.float32 if self.params.out_dtype == VP_OUT_F32 else torch.bfloat16
        t = pl.totals
        return dict(
            pixel_values=torch.empty(t["img_rows"], self.D, dtype=dt, device=self.device),
            pixel_values_videos=torch.empty(t["vid_rows"], self.D, dtype=dt, device=self.device),
            image_grid_thw=torch.empty(t["n_images"], 3, dtype=torch.int64, device=self.device),
            video_grid_thw=torch.empty(t["n_videos"], 3, dtype=torch.int64, device=self.device),
            clip_status=torch.empty(max(pl.n, 1), dtype=torch.int32, device=self.device),
            workspace=resize_workspace(pl.n, self.device),
        )

    # -- H5-H7 --
    def run(self, pl: Plan, frames, clip_byte_offset, row_pitch, out=None, stream=None, strict=True):
        """Strict by default: a clip whose rows the kernels could not write (VP_ECAPACITY,
        VP_EUNSUPPORTED) raises.  Clips with invalid descriptors are recorded as VP_EINVAL in
        ``clip_status`` / the plan without aborting the batch."""
        out = self.alloc_outputs(pl) if out is None else out
        params = self.launch_params(pl)
        resize_normalize_patchify(params, pl.plans_dev, pl.n, frames, clip_byte_offset,
                                  row_pitch, out["pixel_values"] if out["pixel_values"].numel() else None,
                                  out["pixel_values_videos"] if out["pixel_values_videos"].numel() else None,
                                  out["image_grid_thw"], out["video_grid_thw"], out["clip_status"],
                                  workspace=out.get("workspace"), stream=stream)
        if strict:
            st = out["clip_status"][: pl.n].cpu().numpy()
            bad = np.nonzero((st != VP_OK) & (st != VP_EINVAL))[0]
            if len(bad):
                raise VpError(int(st[bad[0]]), f"clip {int(bad[0])}")
        return out

    # -- H8 --
    def rope_index(self, mm_token_type, cu_seqlens, image_grid_thw, video_grid_thw,
                   variant=None, second_per_grid=None, tokens_per_second=None, stream=None,
                   strict=True):
        """vp_rope_index for a packed batch; variant / tokens_per_second default to the preprocessor's (preset)."""
        variant = self.rope_variant if variant is None else variant
        tokens_per_second = self.tokens_per_second if tokens_per_second is None else tokens_per_second
        L = mm_token_type.numel()
        B = cu_seqlens.numel() - 1
        nv = video_grid_thw.shape[0] if video_grid_thw is not None else 0
        pos = torch.empty(3, L, dtype=torch.int64, device=self.device)
        deltas = torch.empty(max(B, 1), dtype=torch.int64, device=self.device)
        st = torch.empty(B + 1, dtype=torch.int32, device=self.device)
        ws = torch.empty(rope_index_workspace_bytes(B, nv), dtype=torch.uint8, device=self.device)
        rope_index(self.params, variant, mm_token_type, cu_seqlens, image_grid_thw, video_grid_thw, pos, deltas,
                   st, ws, second_per_grid, tokens_per_second, stream=stream)
        if strict:
            s = st.cpu().numpy()
            bad = np.nonzero(s[:B])[0]
            if len(bad) or s[B] != VP_OK:
                where = f"sequence {int(bad[0])}" if len(bad) else "batch (visual grids left without placeholders)"
                raise PlacementMismatch(f"placeholder tokens != visual features in {where} (P:165 strict policy)")
        return pos, deltas[:B], st
