"""GPU: vp_plan_records + vp_pack_offsets (H10 device side) against numpy on a simulated 4-rank gather."""
import numpy as np
import pytest
import torch

import oracle as O
import vp_inputs as I

pytestmark = pytest.mark.gpu


def test_records_and_pack_offsets():
    import paper_2604_16893_b200 as vp
    from parity import oracle_params
    params, clips = I.config("cfg4")
    clips = clips + [I.clip(0, 30.0, 64, 64)]                # one invalid clip -> zero record
    world = 4
    clips = (clips * 2)[: 12 * world]
    pre = vp.VisualPreprocessor(**params)
    recs = []
    for r in range(world):
        pl = pre.plan(clips[12 * r: 12 * (r + 1)])
        rec = torch.empty(12 * 4, dtype=torch.int32, device="cuda")
        vp.plan_records(pl.plans_dev, 12, params["merge_size"], rec)
        recs.append(rec)
    g = torch.cat(recs)
    tok = torch.empty(12 * world + 1, dtype=torch.int64, device="cuda")
    pat = torch.empty(12 * world + 1, dtype=torch.int64, device="cuda")
    vp.pack_offsets(g, world, 12, tok, pat)
    torch.cuda.synchronize()
    oplans, _ = O.plan_batch(oracle_params(pre.params), clips)
    ref = np.array([[p.grid[0], p.grid[1], p.grid[2], p.tokens] if p.status == O.VP_OK else [0, 0, 0, 0]
                    for p in oplans], dtype=np.int64)
    assert np.array_equal(g.cpu().numpy().reshape(-1, 4), ref)
    assert tok.cpu().tolist() == np.concatenate([[0], np.cumsum(ref[:, 3])]).tolist()
    assert pat.cpu().tolist() == np.concatenate([[0], np.cumsum(ref[:, 0] * ref[:, 1] * ref[:, 2])]).tolist()
