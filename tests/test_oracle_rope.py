"""Pins for oracle O10-O11 (timestamps, MRoPE ids, strict validation).

* HF Qwen3VLModel.get_rope_index (called unbound on a stub) -- library pin of C18/C21
* text-only sequences reduce to 1-D RoPE arange(L) on all three axes
* HF Qwen2-VL docstring example for the classic time-scaled variant (C19; library code is wrong for t>1)
* HF Qwen3VLProcessor._calculate_timestamps -- library pin of C22
* SPEC S:446-448 strict alignment examples (also in test_oracle_plan)
"""
import types

import numpy as np
import pytest
import torch

import oracle as O
import vp_inputs as I


def _hf_qwen3_rope(seqs, image_grids, video_grids, merge):
    from transformers.models.qwen3_vl.modeling_qwen3_vl import Qwen3VLModel
    stub = types.SimpleNamespace(config=types.SimpleNamespace(
        vision_config=types.SimpleNamespace(spatial_merge_size=merge)))
    stub.get_vision_position_ids = types.MethodType(Qwen3VLModel.get_vision_position_ids, stub)
    B, L = len(seqs), max(len(s) for s in seqs)
    ids = torch.zeros(B, L, dtype=torch.long)
    tt = torch.zeros(B, L, dtype=torch.int)
    am = torch.zeros(B, L, dtype=torch.long)
    for b, s in enumerate(seqs):
        tt[b, :len(s)] = torch.from_numpy(np.asarray(s, dtype=np.int32))
        am[b, :len(s)] = 1
    pos, deltas = Qwen3VLModel.get_rope_index(
        stub, ids, tt,
        torch.tensor(image_grids, dtype=torch.long).reshape(-1, 3) if image_grids else None,
        torch.tensor(video_grids, dtype=torch.long).reshape(-1, 3) if video_grids else None,
        attention_mask=am)
    return [pos[:, b, :len(s)].numpy() for b, s in enumerate(seqs)], deltas[:, 0].tolist()


def _video_runs(grid, merge, ts_len=6):
    t, h, w = grid
    runs = []
    for _ in range(t):       # "<t seconds><vision_start> group <vision_end>" per temporal group
        runs += [(0, ts_len + 1), (2, h * w // merge ** 2), (0, 1)]
    return runs


def _mixed_batch():
    m = 2
    img = [(1, 16, 24), (1, 8, 8), (1, 64, 64)]
    vid = [(4, 8, 8), (3, 12, 20)]
    s0 = [(0, 10)] + _video_runs(vid[0], m) + [(0, 5), (1, 96), (0, 3)]
    s1 = [(0, 4), (1, 16), (0, 2)] + _video_runs(vid[1], m) + [(0, 9)]
    s2 = [(0, 33)]
    s3 = [(0, 64), (1, 1024), (0, 32)]
    return [I.token_types(s) for s in (s0, s1, s2, s3)], [img[0], img[1], img[2]], vid, m


def test_rope_matches_hf_qwen3():
    seqs, img, vid, m = _mixed_batch()
    ours, deltas, st, bst = O.rope_index(seqs, img, vid, m, variant=0)
    ref, ref_d = _hf_qwen3_rope(seqs, img, vid, m)
    assert bst == O.VP_OK and all(s == O.VP_OK for s in st)
    for a, b in zip(ours, ref):
        assert np.array_equal(a, b)
    assert deltas == ref_d


def test_text_only_is_1d_rope():
    L = 57
    ids, deltas, st, _ = O.rope_index([np.zeros(L, np.int8)], [], [], 2)
    assert np.array_equal(ids[0], np.tile(np.arange(L), (3, 1))) and deltas == [0]


def test_time_scaled_variant_docstring_example():
    """HF Qwen2.5-VL get_rope_index docstring: `interval = tokens_per_second * temporal_patch_size / fps`;
    fps 1, tokens_per_second 25, temporal_patch_size 2 -> llm grid 3x2x2 has
    T [0,0,0,0,50,50,50,50,100,...], H [0,0,1,1,...], W [0,1,0,1,...].  The interval comes from the oracle's
    own chain second_per_grid(tp, fps) -> qwen25_interval, not from the test."""
    spg = O.second_per_grid(2, 1.0)
    assert spg == 2.0 and O.qwen25_interval(25, spg) == 50
    ids, deltas, st, _ = O.rope_index([np.full(12, 2)], [], [(3, 4, 4)], 2, variant=2,
                                      second_per_grid_ts=[spg], tokens_per_second=25)
    assert ids[0][0].tolist() == [0] * 4 + [50] * 4 + [100] * 4
    assert ids[0][1].tolist() == [0, 0, 1, 1] * 3
    assert ids[0][2].tolist() == [0, 1, 0, 1] * 3
    assert deltas == [101 - 12] and st == [O.VP_OK]


def test_classic_variant_is_unit_interval():
    """QWEN2 classic (C19): consecutive temporal grids one id apart; equals QWEN25 with tps*int(spg) = 1."""
    a, da, _, _ = O.rope_index([np.full(12, 2)], [], [(3, 4, 4)], 2, variant=1)
    assert a[0][0].tolist() == [0] * 4 + [1] * 4 + [2] * 4 and da == [3 - 12]
    b, db, _, _ = O.rope_index([np.full(12, 2)], [], [(3, 4, 4)], 2, variant=2, second_per_grid_ts=[1.9],
                               tokens_per_second=1)
    assert np.array_equal(a[0], b[0]) and da == db


def test_qwen25_interval_matches_hf():
    """Library pin of the interval rule: HF Qwen2_5_VLModel.get_rope_index called unbound on a stub whose
    get_vision_position_ids records the time_interval it is handed (its own id formula is not used: it is
    wrong for t > 1 in the installed version), and Qwen2_5_VLProcessor's second_per_grid_ts = tp / fps."""
    from transformers.models.qwen2_5_vl.modeling_qwen2_5_vl import Qwen2_5_VLModel
    seen = []

    def fake_vpi(self, start, grid, tms, sms, time_interval, device=None):
        seen.append(time_interval)
        n = int(grid[0]) * int(grid[1]) // sms * int(grid[2]) // sms
        return torch.zeros(3, n, dtype=torch.long)

    stub = types.SimpleNamespace(config=types.SimpleNamespace(
        vision_config=types.SimpleNamespace(spatial_merge_size=2, tokens_per_second=25)))
    stub.get_vision_position_ids = types.MethodType(fake_vpi, stub)
    fps_list = [1.0, 2.0, 1.5, 0.5, 3.0, 2.0 / 3.0, 0.7, 29.97]
    spg = [2 / f for f in fps_list]
    grids = torch.tensor([[1, 4, 4]] * len(spg))
    types_ = []
    for _ in spg:
        types_ += [0, 0] + [2] * 4
    tt = torch.tensor([types_])
    Qwen2_5_VLModel.get_rope_index(stub, torch.zeros_like(tt), tt, None, grids, torch.tensor(spg, dtype=torch.float64))
    assert seen == [O.qwen25_interval(25, O.second_per_grid(2, f)) for f in fps_list]
    assert seen == [50, 25, 25, 100, 0, 75, 50, 0]        # truncation toward zero: 1.33 -> 1, 0.667 -> 0


def test_rope_run_invariants():
    seqs, img, vid, m = _mixed_batch()
    ids, deltas, _, _ = O.rope_index(seqs, img, vid, m)
    for s, a in zip(seqs, ids):
        # text ids are consecutive on all three axes; every run starts above all earlier ids
        k, prev_max = 0, -1
        while k < len(s):
            e = k
            while e < len(s) and s[e] == s[k]:
                e += 1
            run = a[:, k:e]
            assert run.min() == prev_max + 1
            if s[k] == 0:
                assert np.array_equal(run, np.tile(np.arange(prev_max + 1, prev_max + 1 + e - k), (3, 1)))
            prev_max = run.max()
            k = e


def test_strict_mismatch_detection():
    """P:165 strict failure; S:444 names sample and both counts.  Off-by-one runs, a missing grid,
    adjacent video groups without separating text, and leftover grids."""
    m = 2
    g = (1, 8, 8)                                           # 16 tokens
    ok = I.token_types([(0, 3), (1, 16), (0, 2)])
    short = I.token_types([(0, 3), (1, 15), (0, 2)])
    _, _, st, bst = O.rope_index([ok, short], [g, g], [], m)
    assert st == [O.VP_OK, O.VP_EMISMATCH] and bst == O.VP_OK
    _, _, st, bst = O.rope_index([ok, ok], [g], [], m)      # second run has no grid
    assert st == [O.VP_OK, O.VP_EMISMATCH]
    _, _, st, bst = O.rope_index([ok], [g, g], [], m)       # leftover grid
    assert st == [O.VP_OK] and bst == O.VP_EMISMATCH
    merged = I.token_types([(0, 3), (2, 32), (0, 2)])      # two t=1 groups glued together
    _, _, st, _ = O.rope_index([merged], [], [(2, 8, 8)], m)
    assert st == [O.VP_EMISMATCH]


def test_timestamps_match_hf():
    from transformers.models.qwen3_vl.processing_qwen3_vl import Qwen3VLProcessor
    for total, fps, mx in [(1800, 30.0, 64), (100, 10.0, 128), (7, 29.97, 64), (108000, 30.0, 768), (1, 24.0, 8)]:
        n, idx = O.sample_frame_indices(total, fps, 2.0, mx, 2)
        ref = Qwen3VLProcessor._calculate_timestamps(None, list(idx), fps, 2)
        assert O.group_timestamps(idx, fps, 2) == ref
    # closed form: S:81 indices [2,7,...,97] at 10 fps -> groups (0.2+0.7)/2, (1.2+1.7)/2, ...
    n, idx = O.sample_frame_indices(100, 10.0, 2.0, 128, 2)
    assert O.group_timestamps(idx, 10.0, 2) == pytest.approx([0.45 + g for g in range(10)])
