"""ctypes loader for libvp.so (the C ABI in include/vp.h).  Argument marshalling only.

There is no CPU fallback: if libvp.so is missing this module raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libvp.so")

# vp_status
VP_OK, VP_EINVAL, VP_EALIGN, VP_EMISMATCH, VP_ECAPACITY, VP_ECUDA, VP_EUNSUPPORTED = range(7)
VP_ROPE_QWEN3_SPLIT, VP_ROPE_QWEN2, VP_ROPE_QWEN25 = 0, 1, 2
VP_SAMPLE_CENTER_BIN, VP_SAMPLE_LINSPACE = 0, 1
VP_RESIZE_FLOAT, VP_RESIZE_U8 = 0, 1
VP_OUT_BF16, VP_OUT_F32 = 0, 1
VP_BUDGET_PER_FRAME, VP_BUDGET_TOTAL = 0, 1
VP_SYNTH_RAMP, VP_SYNTH_NOISE = 0, 1

# totals[] indices (vp.h)
TOT = dict(indices=0, img_rows=1, vid_rows=2, img_tokens=3, vid_tokens=4, n_images=5, n_videos=6,
           vid_groups=7, tiles=8, flags=9, n_invalid=10, variants=11)
TOT_LEN = 12

EXPORTED = ["vp_plan_frames", "vp_resize_workspace_bytes", "vp_resize_normalize_patchify", "vp_rope_index_workspace_bytes", "vp_rope_index",
            "vp_pack_offsets", "vp_plan_records", "vp_synth_frames", "vp_status_string", "vp_last_error_detail",
            "vp_abi_version", "vp_struct_sizes", "vp_dedup_clips", "vp_dedup_views",
            "vp_plan_second_per_grid", "vp_nv12_to_rgb", "vp_vision_ids_workspace_bytes", "vp_vision_ids"]


class VpParams(C.Structure):
    _fields_ = [("target_fps", C.c_double), ("max_frames", C.c_int32), ("temporal_patch_size", C.c_int32),
                ("patch_size", C.c_int32), ("merge_size", C.c_int32), ("video_max_pixels", C.c_int64),
                ("image_max_pixels", C.c_int64), ("min_pixels", C.c_int64), ("budget_mode", C.c_int32),
                ("sampling", C.c_int32), ("mean", C.c_double * 3), ("std", C.c_double * 3),
                ("out_dtype", C.c_int32), ("launch_mask", C.c_int32),
                ("min_frames", C.c_int32), ("resize_mode", C.c_int32)]


DESC_DTYPE = np.dtype([("total_source_frames", "<i8"), ("source_fps", "<f8"), ("height", "<i4"),
                       ("width", "<i4"), ("is_image", "<i4"), ("pad_", "<i4")])
PLAN_DTYPE = np.dtype([("status", "<i4"), ("is_image", "<i4"), ("in_h", "<i4"), ("in_w", "<i4"),
                       ("n_frames", "<i4"), ("out_h", "<i4"), ("out_w", "<i4"), ("grid_t", "<i4"),
                       ("grid_h", "<i4"), ("grid_w", "<i4"), ("index_offset", "<i8"), ("patch_offset", "<i8"),
                       ("token_offset", "<i8"), ("grid_index", "<i8"), ("group_offset", "<i8"),
                       ("tile_offset", "<i8"), ("tile_count", "<i4"), ("kernel_variant", "<i4"),
                       ("effective_fps", "<f8")])


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2604_16893_b200/_build.py` "
                          f"(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    i32, i64, u64, sz = C.c_int32, C.c_int64, C.c_uint64, C.c_size_t
    P = C.POINTER(VpParams)
    sig = {
        "vp_plan_frames": (i32, [P, vp, i32, vp, vp, i64, vp, i64, vp, vp]),
        "vp_resize_workspace_bytes": (sz, [i32]),
        "vp_resize_normalize_patchify": (i32, [P, vp, i32, vp, vp, vp, vp, i64, vp, i64, vp, vp, vp, vp, sz, vp]),
        "vp_rope_index_workspace_bytes": (sz, [i32, i32]),
        "vp_rope_index": (i32, [P, i32, vp, vp, i32, i64, vp, i32, vp, i32, vp, i32, vp, vp, vp, vp, sz, vp]),
        "vp_pack_offsets": (i32, [vp, i32, i32, vp, vp, vp]),
        "vp_plan_records": (i32, [vp, i32, i32, vp, vp]),
        "vp_synth_frames": (i32, [i32, u64, vp, i32, i32, i32, i64, vp, vp]),
        "vp_status_string": (C.c_char_p, [i32]),
        "vp_last_error_detail": (C.c_char_p, []),
        "vp_abi_version": (i32, []),
        "vp_struct_sizes": (i32, []),
        "vp_dedup_clips": (i32, [vp, i32, vp, vp, vp, vp]),
        "vp_dedup_views": (i32, [vp, vp, i32, vp, vp, vp, vp]),
        "vp_plan_second_per_grid": (i32, [vp, vp, i32, i32, vp, vp]),
        "vp_nv12_to_rgb": (i32, [vp, vp, i64, i64, i32, i32, i32, vp, i64, i64, vp]),
        "vp_vision_ids_workspace_bytes": (sz, [i32]),
        "vp_vision_ids": (i32, [vp, i32, i32, vp, vp, vp, sz, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    sizes = lib.vp_struct_sizes()
    got = (sizes & 1023, (sizes >> 10) & 1023, (sizes >> 20) & 1023)
    want = (C.sizeof(VpParams), DESC_DTYPE.itemsize, PLAN_DTYPE.itemsize)
    if got != want:
        raise ImportError(f"libvp struct layout mismatch: library {got}, binding {want}")
    return lib


lib = _load()


class VpError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        detail = lib.vp_last_error_detail().decode(errors="replace")
        super().__init__(f"{what}: {lib.vp_status_string(status).decode()} ({detail})")


def check(status: int, what: str) -> None:
    if status != VP_OK:
        raise VpError(status, what)
