"""N2 -- model-family presets ("natively supports the Qwen2-VL, Qwen2.5-VL, Qwen3-VL, and Qwen3.5 series";
P:268).  Data only: the vision-side constants of each family (patch / merge / temporal patch sizes, normalisation
mean and std, MRoPE variant, time scale) with the paper's training budgets (2 fps, <= 128 frames, 262,144
pixels per video frame, 1,048,576 per image).  The kernels are the same for every family; only the parameters and
the vp_rope_index variant differ.

Sources (pinned in tests/test_oracle_presets.py against the installed HF processors / configs):
  Qwen2-VL   : patch 14, merge 2, temporal 2, OpenAI-CLIP mean/std, classic MRoPE (temporal id step 1).
  Qwen2.5-VL : as Qwen2-VL, time-scaled temporal ids: step = tokens_per_second * int(second_per_grid_ts),
               second_per_grid_ts = temporal_patch_size / sampled fps (vp_plan_second_per_grid); tokens_per_second
               is the HF Qwen2_5_VLVisionConfig default (4); a checkpoint's config.json value overrides it
               (VisualPreprocessor.from_preset("qwen2_5_vl", tokens_per_second=...)).
  Qwen3-VL   : patch 16, merge 2, temporal 2, mean = std = 0.5, videos split into per-frame-group grids
               separated by timestamp text (VP_ROPE_QWEN3_SPLIT, C18).
  Qwen3.5    : the Qwen3-VL vision preprocessing and split MRoPE (HF Qwen3_5Model.get_rope_index).
"""
from __future__ import annotations

from ._lib import VP_ROPE_QWEN2, VP_ROPE_QWEN3_SPLIT, VP_ROPE_QWEN25

OPENAI_CLIP_MEAN = (0.48145466, 0.4578275, 0.40821073)
OPENAI_CLIP_STD = (0.26862954, 0.26130258, 0.27577711)
_PAPER_BUDGETS = dict(target_fps=2.0, max_frames=128, video_max_pixels=262144, image_max_pixels=1048576)

PRESETS = {
    "qwen2_vl": dict(patch_size=14, merge_size=2, temporal_patch_size=2, mean=OPENAI_CLIP_MEAN, std=OPENAI_CLIP_STD,
                     rope_variant=VP_ROPE_QWEN2, tokens_per_second=0),
    "qwen2_5_vl": dict(patch_size=14, merge_size=2, temporal_patch_size=2, mean=OPENAI_CLIP_MEAN,
                       std=OPENAI_CLIP_STD, rope_variant=VP_ROPE_QWEN25, tokens_per_second=4),
    "qwen3_vl": dict(patch_size=16, merge_size=2, temporal_patch_size=2, mean=(0.5, 0.5, 0.5), std=(0.5, 0.5, 0.5),
                     rope_variant=VP_ROPE_QWEN3_SPLIT, tokens_per_second=0),
    "qwen3_5": dict(patch_size=16, merge_size=2, temporal_patch_size=2, mean=(0.5, 0.5, 0.5), std=(0.5, 0.5, 0.5),
                    rope_variant=VP_ROPE_QWEN3_SPLIT, tokens_per_second=0),
}


def preset(name: str, **overrides) -> tuple[dict, dict]:
    """(vp_params keyword arguments, MRoPE settings {rope_variant, tokens_per_second}) of a model family, with the
    paper's budgets; keyword overrides replace either."""
    if name not in PRESETS:
        raise KeyError(f"unknown preset {name!r}; one of {sorted(PRESETS)}")
    p = dict(_PAPER_BUDGETS)
    p.update(PRESETS[name])
    p.update(overrides)
    rope = {"rope_variant": p.pop("rope_variant"), "tokens_per_second": p.pop("tokens_per_second")}
    return p, rope
