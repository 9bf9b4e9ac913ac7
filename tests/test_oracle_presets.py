"""N2 pins (CPU): the model-family presets (paper_2604_16893_b200/presets.py) against the installed HF
processors and configs, the Qwen3.5 MRoPE convention against HF Qwen3_5Model.get_rope_index (it equals the
oracle's Qwen3-VL split variant), and the Qwen2.5-VL time scale against HF VideoMetadata.sampled_fps."""
import types

import numpy as np
import torch

import oracle as O
import vp_inputs as I


def test_presets_match_hf_processors():
    from paper_2604_16893_b200.presets import PRESETS
    from paper_2604_16893_b200 import VP_ROPE_QWEN2, VP_ROPE_QWEN25, VP_ROPE_QWEN3_SPLIT
    from transformers.models.qwen2_vl.image_processing_qwen2_vl import Qwen2VLImageProcessor
    from transformers.models.qwen3_vl.video_processing_qwen3_vl import Qwen3VLVideoProcessor
    from transformers.models.qwen2_5_vl.configuration_qwen2_5_vl import Qwen2_5_VLVisionConfig
    from transformers.models.qwen3_5.configuration_qwen3_5 import Qwen3_5VisionConfig
    q2 = Qwen2VLImageProcessor()
    for name in ("qwen2_vl", "qwen2_5_vl"):
        p = PRESETS[name]
        assert (p["patch_size"], p["merge_size"], p["temporal_patch_size"]) == (q2.patch_size, q2.merge_size,
                                                                                q2.temporal_patch_size)
        assert np.allclose(p["mean"], q2.image_mean, atol=0, rtol=0) and np.allclose(p["std"], q2.image_std, 0, 0)
    assert PRESETS["qwen2_5_vl"]["tokens_per_second"] == Qwen2_5_VLVisionConfig().tokens_per_second
    q3 = Qwen3VLVideoProcessor()
    for name in ("qwen3_vl", "qwen3_5"):
        p = PRESETS[name]
        assert (p["patch_size"], p["merge_size"], p["temporal_patch_size"]) == (q3.patch_size, q3.merge_size,
                                                                                q3.temporal_patch_size)
        assert tuple(p["mean"]) == tuple(q3.image_mean) and tuple(p["std"]) == tuple(q3.image_std)
    c35 = Qwen3_5VisionConfig()
    assert (c35.patch_size, c35.spatial_merge_size, c35.temporal_patch_size) == (16, 2, 2)
    assert PRESETS["qwen2_vl"]["rope_variant"] == VP_ROPE_QWEN2
    assert PRESETS["qwen2_5_vl"]["rope_variant"] == VP_ROPE_QWEN25
    assert PRESETS["qwen3_vl"]["rope_variant"] == PRESETS["qwen3_5"]["rope_variant"] == VP_ROPE_QWEN3_SPLIT


def test_qwen35_rope_is_the_split_variant():
    """HF Qwen3_5Model.get_rope_index (unbound on a stub) == oracle variant 0 on a mixed batch."""
    from transformers.models.qwen3_5.modeling_qwen3_5 import Qwen3_5Model
    m = 2
    seqs, img, vid = [], [], []
    img.append((1, 8, 12))
    seqs.append(I.token_types([(0, 5), (1, 24), (0, 3)]))
    vid.append((3, 6, 8))
    runs = [(0, 4)]
    for _ in range(3):
        runs += [(0, 6), (2, 12), (0, 1)]
    seqs.append(I.token_types(runs + [(0, 2)]))
    stub = types.SimpleNamespace(config=types.SimpleNamespace(vision_config=types.SimpleNamespace(spatial_merge_size=m)))
    stub.get_vision_position_ids = types.MethodType(Qwen3_5Model.get_vision_position_ids, stub)
    B, L = len(seqs), max(len(s) for s in seqs)
    tt = torch.zeros(B, L, dtype=torch.int)
    am = torch.zeros(B, L, dtype=torch.long)
    for b, s in enumerate(seqs):
        tt[b, :len(s)] = torch.from_numpy(np.asarray(s, dtype=np.int32))
        am[b, :len(s)] = 1
    pos, deltas = Qwen3_5Model.get_rope_index(stub, torch.zeros(B, L, dtype=torch.long), tt,
                                              torch.tensor(img), torch.tensor(vid), attention_mask=am)
    ids, od, st, bst = O.rope_index(seqs, img, vid, m, variant=0)
    for b, s in enumerate(seqs):
        assert np.array_equal(pos[:, b, :len(s)].numpy(), ids[b])
    assert deltas[:, 0].tolist() == od


def test_sampled_fps_is_hf_order():
    """Qwen2.5 time scale input: oracle hf_sampled_fps == HF VideoMetadata.sampled_fps bit for bit (n / total * fps),
    so second_per_grid = tp / sampled_fps and int() of it agree with the processor's second_per_grid_ts."""
    import random
    from transformers.video_utils import VideoMetadata
    rng = random.Random(1)
    for _ in range(2000):
        total = rng.randint(1, 200000)
        fps = rng.choice([23.976, 24.0, 25.0, 29.97, 30.0, 59.94, rng.uniform(0.2, 240)])
        n, idx = O.sample_frame_indices(total, fps, 2.0, 128, 2)
        md = VideoMetadata(total_num_frames=total, fps=fps, frames_indices=idx)
        assert O.hf_sampled_fps(n, total, fps) == md.sampled_fps
        assert O.second_per_grid(2, md.sampled_fps) == 2 / md.sampled_fps
