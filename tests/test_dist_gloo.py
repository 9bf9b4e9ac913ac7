"""world_size-2 gloo tests of the N>1 host path (H10): contiguous clip sharding + all-gather of per-clip
(t,h,w,tokens) records gives every rank the same global token/patch offsets as a single-process run.
The device-side scan (vp_pack_offsets) is checked against numpy in tests/test_gpu_dist.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import vp_inputs as I


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _records(params, clips):
    plans, _ = O.plan_batch(params, clips)
    m = params["merge_size"]
    return np.array([[p.grid[0], p.grid[1], p.grid[2], p.tokens] if p.status == O.VP_OK else [0, 0, 0, 0]
                     for p in plans], dtype=np.int32).reshape(-1)


def _worker(rank, world, port, clips_per_rank, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_16893_b200.dist import gather_records, shard_range
    params, clips = I.config("cfg4")
    clips = (clips * 4)[: clips_per_rank * world]
    a, b = shard_range(len(clips), world, rank)
    rec = torch.from_numpy(_records(params, clips[a:b]))
    g = gather_records(rec).numpy().reshape(-1, 4)
    tok = np.concatenate([[0], np.cumsum(g[:, 3].astype(np.int64))])
    q.put((rank, g.tolist(), tok.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gather_and_offsets_match_single_process(world):
    clips_per_rank = 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, clips_per_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    params, clips = I.config("cfg4")
    clips = (clips * 4)[: clips_per_rank * world]
    ref = _records(params, clips).reshape(-1, 4)
    ref_tok = np.concatenate([[0], np.cumsum(ref[:, 3].astype(np.int64))])
    for rank, g, tok in res:
        assert np.array_equal(np.array(g), ref), rank
        assert tok == ref_tok.tolist()


def test_shard_range_covers_exactly_once():
    from paper_2604_16893_b200.dist import shard_range
    for n in (0, 1, 7, 512, 513):
        for w in (1, 2, 3, 4, 8):
            seen = []
            for r in range(w):
                a, b = shard_range(n, w, r)
                seen += list(range(a, b))
                assert b - a in (n // w, n // w + 1)
            assert seen == list(range(n))


@pytest.mark.parametrize("world", [2, 4])
def test_bench_launcher_spawns_ranks(world):
    """`python bench.py --gpus N` outside torchrun re-executes itself through torch.distributed.run (one process per
    rank, rendezvous on 127.0.0.1); --dist-selftest runs the N>1 plumbing of the bench on gloo: the cfg5 clip shards,
    the all-gather of per-clip int32 records in rank order and the max-over-ranks reduction of the step time."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", str(world), "--backend", "gloo",
                        "--dist-selftest"], capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    d = json.loads(line)
    assert d["dist_selftest"] == "ok" and d["world"] == world and d["gathered_records"] == 512
    assert d["max_over_ranks"] == world
