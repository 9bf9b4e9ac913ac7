"""N4 oracle pins (CPU): NV12 -> RGB against OpenCV's COLOR_YUV2RGB_NV12 (the decoder-side conversion it restates),
and the vision-tower patch ids / cu_seqlens against HF Qwen3-VL's rot_pos_emb (called on a stub whose rotary table
is the identity, so its embedding lookup returns the ids) and its cu_seqlens expression."""
import types

import numpy as np
import torch

import oracle as O


def test_nv12_matches_opencv():
    import cv2
    rng = np.random.default_rng(0)
    for H, W in ((2, 2), (6, 10), (32, 48), (70, 126)):
        for kind in ("uniform", "extreme"):
            if kind == "uniform":
                yuv = rng.integers(0, 256, (H * 3 // 2, W), dtype=np.uint8)
            else:                                   # saturating corners: Y, U, V in {0, 16, 128, 235, 240, 255}
                yuv = rng.choice(np.array([0, 16, 128, 235, 240, 255], np.uint8), (H * 3 // 2, W))
            ref = cv2.cvtColor(yuv, cv2.COLOR_YUV2RGB_NV12)
            got = O.nv12_to_rgb(yuv[:H], yuv[H:])
            assert np.array_equal(got, ref), (H, W, kind)


def test_vision_ids_match_hf():
    from transformers.models.qwen3_vl.modeling_qwen3_vl import Qwen3VLVisionModel
    grids = [(1, 4, 6), (3, 8, 4), (2, 2, 2), (1, 16, 12)]
    stub = types.SimpleNamespace(spatial_merge_size=2)
    stub.rotary_pos_emb = lambda n: torch.arange(n, dtype=torch.float64).reshape(-1, 1)   # table row i = [i]
    emb = Qwen3VLVisionModel.rot_pos_emb(stub, torch.tensor(grids))
    assert np.array_equal(emb.numpy().astype(np.int64), O.vision_pos_ids(grids, 2))
    g = torch.tensor(grids)
    cu = torch.nn.functional.pad(torch.repeat_interleave(g[:, 1] * g[:, 2], g[:, 0]).cumsum(0), (1, 0))
    assert cu.tolist() == O.vision_cu_seqlens(grids)
