#!/usr/bin/env python
"""Bench of the B200 visual-preprocessing hot path (EasyVideoR1, arXiv 2604.16893).

Metric (BASELINE.json): visual tokens/s (t*h*w/m^2) and achieved HBM GB/s vs peak.
Workload (N=1 default): cfg5 -- the GRPO rollout batch of 512 clips shaped like cfg2 (30 fps
1280x720 source, 2 fps, <=64 frames, 262,144 px/frame -> 384x672, grid (32,24,42), 8,064 tokens
each), sharded by clip over the ranks (strong scaling: the job is always 512 clips).

One step = the whole hot path for the rank's clips, all on the device:
  K1 vp_plan_frames -> K3 vp_resize_normalize_patchify -> K4 vp_rope_index
  (+ N>1: vp_plan_records -> NCCL all_gather (torch.distributed) -> vp_pack_offsets).
Inputs are synthetic u8 frames written into HBM by vp_synth_frames before timing (90.6 GB at N=1,
larger than L2, so no L2 flush is needed).  `e2e` times the same path from pinned HOST frames,
the host->device copies inside the timed region, pipelined clip-chunk by clip-chunk.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--clips C]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "visual tokens/sec and achieved HBM GB/s vs peak at 1/2/4/8 B200"
UNIT = "visual tokens/s"
JOB_CLIPS = 512
CLOCK_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")


def cfg5_clip():
    import vp_inputs as I
    return I.clip(1800, 30.0, 720, 1280)


def cfg5_params():
    import vp_inputs as I
    return I.qwen3_params(max_frames=64)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={CLOCK_FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as g:
            for line in g:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------------------------

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2604_16893_b200 as vp
    import vp_inputs as I
    from paper_2604_16893_b200.dist import gather_records_async

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if args.config == "cfg5":
        job_clips = args.clips if args.clips else JOB_CLIPS
        params, all_clips = cfg5_params(), [cfg5_clip()] * job_clips
    else:                                   # other BASELINE configs (profiling / reporting only)
        params, all_clips = I.config(args.config)
        job_clips = len(all_clips)
    from paper_2604_16893_b200.dist import shard_range
    assert job_clips % world == 0, "clips must divide evenly over ranks"
    a, b = shard_range(job_clips, world, rank)
    clips = all_clips[a:b]
    per = len(clips)
    pre = vp.VisualPreprocessor(device=dev, **params)
    m = pre.params.merge_size

    # ---------------- setup (untimed) ----------------
    pl = pre.plan(clips)
    P = pre.launch_params(pl)              # params + the plan's kernel-variant launch hint
    ph = pl.plans_host
    off, pitch, total_bytes = pre.frames_layout(pl)
    frames = torch.empty(total_bytes, dtype=torch.uint8, device=dev)
    idx_host = pl.frame_indices.cpu().numpy()
    for k in range(per):
        n, H, W = int(ph["n_frames"][k]), int(ph["in_h"][k]), int(ph["in_w"][k])
        ids = torch.from_numpy(idx_host[ph["index_offset"][k]: ph["index_offset"][k] + n].copy()).to(dev)
        vp.synth_frames(vp.VP_SYNTH_NOISE, 1000003 * 0 + rank * per + k, ids, H, W, frames[off[k]:], int(pitch[k]))
    off_d = torch.from_numpy(off).to(dev)
    pitch_d = torch.from_numpy(pitch).to(dev)
    out = pre.alloc_outputs(pl)            # includes the K3 workspace (caller-owned scratch)
    # token-type sequences: one sequence per clip (Qwen3-VL: "<t s><vision_start> group <vision_end>" per group)
    seqs = []
    for k in range(per):
        gt, gh, gw = int(ph["grid_t"][k]), int(ph["grid_h"][k]), int(ph["grid_w"][k])
        runs = [(0, 64)]
        if ph["is_image"][k]:
            runs += [(0, 1), (1, gh * gw // (m * m)), (0, 1)]
        else:
            for _ in range(gt):
                runs += [(0, 7), (2, gh * gw // (m * m)), (0, 1)]
        runs.append((0, 32))
        seqs.append(I.token_types(runs))
    n_img = int(pl.totals["n_images"])
    tt = torch.from_numpy(np.concatenate(seqs)).to(dev)
    cu = torch.tensor(np.concatenate([[0], np.cumsum([len(s) for s in seqs])]), dtype=torch.int64, device=dev)
    L = tt.numel()
    pos = torch.empty(3, L, dtype=torch.int64, device=dev)
    deltas = torch.empty(per, dtype=torch.int64, device=dev)
    rst = torch.empty(per + 1, dtype=torch.int32, device=dev)
    ws = torch.empty(vp.rope_index_workspace_bytes(per, per), dtype=torch.uint8, device=dev)
    records = torch.empty(per * 4, dtype=torch.int32, device=dev)
    tok_off = torch.empty(world * per + 1, dtype=torch.int64, device=dev)
    pat_off = torch.empty(world * per + 1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)

    tokens_rank = int(pl.totals["vid_tokens"] + pl.totals["img_tokens"])
    in_bytes = int(sum(int(ph["n_frames"][k]) * int(ph["in_h"][k]) * 3 * int(ph["in_w"][k]) for k in range(per)))
    out_bytes = int((pl.totals["vid_rows"] + pl.totals["img_rows"]) * pre.D * (4 if P.out_dtype else 2))
    k3_bytes = in_bytes + out_bytes

    ev_k3 = []

    def step(record=False):
        vp.plan_frames(P, pl.clips_dev, per, pl.plans_dev, pl.frame_indices, pl.totals_dev, pl.group_timestamps)
        if world > 1:                                          # H10: NCCL all-gather of (t,h,w,tokens) ...
            vp.plan_records(pl.plans_dev, per, m, records)
            gathered, work = gather_records_async(records)     # ... on NCCL's stream, overlapping K3
        if record:
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
        vp.resize_normalize_patchify(P, pl.plans_dev, per, frames, off_d, pitch_d,
                                     out["pixel_values"] if n_img else None,
                                     out["pixel_values_videos"], out["image_grid_thw"], out["video_grid_thw"],
                                     out["clip_status"], workspace=out["workspace"])
        if record:
            b.record(stream)
            ev_k3.append((a, b))
        vp.rope_index(P, vp.VP_ROPE_QWEN3_SPLIT, tt, cu, out["image_grid_thw"] if n_img else None,
                      out["video_grid_thw"], pos, deltas, rst, ws)
        if world > 1:
            work.wait()                                        # the compute stream waits for the gather here
            vp.pack_offsets(gathered, world, per, tok_off, pat_off)

    launches_per_step = k3_launches(int(pl.totals["variants"]), per) + 4 + (2 if world > 1 else 0)   # + K1 (2), K4 (2)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    st = out["clip_status"][:per].cpu().numpy()
    assert (st == 0).all(), f"clip status {np.unique(st)}"
    rs = rst.cpu().numpy()
    assert (rs == 0).all(), "rope status mismatch"
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank) if rank == 0 else None
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step(record=True)
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if clocks else None
    ms_total = t0.elapsed_time(t1)
    k3_ms = float(np.mean([a.elapsed_time(b) for a, b in ev_k3]))
    ms_step = ms_total / args.steps
    t = torch.tensor([ms_step, k3_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step, k3_ms = t.tolist()

    # ---------------- e2e: pinned host frames -> device inside the timed region ----------------
    e2e = None
    if not args.no_e2e and args.config == "cfg5":
        e2e = run_e2e(args, pre, pl, frames, off, pitch, out, tt, cu, pos, deltas, rst, ws, per, dev, world,
                      tokens_rank)

    e2e_nv12 = None
    if not args.no_e2e and args.config == "cfg5":
        e2e_nv12 = run_e2e_nv12(args, pre, pl, frames, off, pitch, out, tt, cu, pos, deltas, rst, ws, per, dev,
                                world, tokens_rank)

    # ---------------- N3: the same job with GRPO dedup (64 prompts x 8 rollouts, P:73 / P:271) ----------------
    dedup = None
    if not args.no_dedup and args.config == "cfg5":
        dedup = run_dedup(args, pre, pl, frames, off_d, pitch_d, tt, cu, pos, deltas, rst, ws, per, a, dev, world,
                          tokens_rank)

    result = None
    if rank == 0:
        peak, peak_src = peaks()
        achieved = k3_bytes / (k3_ms * 1e-3) / 1e9
        tokens_job = tokens_rank * world
        traffic = load_traffic(per)
        result = {
            "metric": METRIC, "value": tokens_job / (ms_step * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": (f"cfg5: GRPO rollout batch of {job_clips} clips (cfg2-shaped: 30 fps 1280x720, "
                                    f"2 fps, <=64 frames, 262144 px/frame -> 384x672, grid (32,24,42)) sharded by "
                                    f"clip over {world} rank(s)") if args.config == "cfg5" else
                                   f"{args.config} (BASELINE.json configs[{args.config[-1]}]), {job_clips} clips",
                       "clips_per_rank": per, "tokens_per_step": tokens_job,
                       "out_dtype": "bf16" if P.out_dtype == 0 else "f32", "model_preset": "Qwen3-VL p16 m2 tp2",
                       "l2": "inputs (%.1f GB/rank) larger than L2, no flush" % (in_bytes / 1e9),
                       "parallelism": f"clip-sharded dp{world}"},
            "hbm_gbs_step": k3_bytes / (ms_step * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": "vp_resize_normalize_patchify (K3: resize_team_kernel, fused AA-bicubic resize/normalise/patchify)",
                         "k3_ms": k3_ms, "algorithmic_bytes_per_launch": k3_bytes, "peak_source": peak_src},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk,
            "e2e": e2e,
            "e2e_nv12": e2e_nv12,
            "dedup_64x8": dedup,
        }
    return result


SIDE_CONFIGS = ("cfg1", "cfg2", "cfg3", "cfg4", "res480p", "res1080p", "res1440p", "res2160p")


def measure_side(name: str, dev, steps: int = 10, warmup: int = 3):
    """One BASELINE config (cfg1-cfg4) or source resolution (16 clips at the cfg2 budget) through K1 + K3 + K4 on
    rank 0: ms per step, visual tokens/s, K3 event time and its HBM fraction, the kernel variants it took."""
    import torch
    import paper_2604_16893_b200 as vp
    import vp_inputs as I
    params, clips = I.config(name)
    pre = vp.VisualPreprocessor(device=dev, **params)
    pl = pre.plan(clips)
    P = pre.launch_params(pl)
    ph = pl.plans_host
    off, pitch, total = pre.frames_layout(pl)
    frames = torch.empty(max(total, 16), dtype=torch.uint8, device=dev)
    idx = pl.frame_indices.cpu().numpy()
    for k in range(pl.n):
        n = int(ph["n_frames"][k])
        ids = torch.from_numpy(idx[ph["index_offset"][k]: ph["index_offset"][k] + n].copy()).to(dev)
        vp.synth_frames(vp.VP_SYNTH_NOISE, 7919 * k + 1, ids, int(ph["in_h"][k]), int(ph["in_w"][k]),
                        frames[int(off[k]):], int(pitch[k]))
    off_d, pitch_d = torch.from_numpy(off).to(dev), torch.from_numpy(pitch).to(dev)
    out = pre.alloc_outputs(pl)
    n_img = int(pl.totals["n_images"])
    stream = torch.cuda.current_stream(dev)
    ev = []

    def step(rec=False):
        vp.plan_frames(P, pl.clips_dev, pl.n, pl.plans_dev, pl.frame_indices, pl.totals_dev, pl.group_timestamps)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        vp.resize_normalize_patchify(P, pl.plans_dev, pl.n, frames, off_d, pitch_d,
                                     out["pixel_values"] if n_img else None,
                                     out["pixel_values_videos"] if pl.totals["vid_rows"] else None,
                                     out["image_grid_thw"], out["video_grid_thw"], out["clip_status"],
                                     workspace=out["workspace"])
        b.record(stream)
        if rec:
            ev.append((a, b))

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    assert (out["clip_status"][: pl.n].cpu().numpy() == 0).all()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        step(True)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    k3 = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    in_b = sum(int(ph["n_frames"][k]) * int(ph["in_h"][k]) * 3 * int(ph["in_w"][k]) for k in range(pl.n)
               if ph["status"][k] == 0)
    out_b = (pl.totals["vid_rows"] + pl.totals["img_rows"]) * pre.D * 2
    peak, _ = peaks()
    tokens = pl.totals["vid_tokens"] + pl.totals["img_tokens"]
    res = {"ms_per_step": ms, "tokens_per_s": tokens / (ms * 1e-3), "k3_ms": k3,
           "k3_gbs": (in_b + out_b) / (k3 * 1e-3) / 1e9, "k3_frac": (in_b + out_b) / (k3 * 1e-3) / 1e9 / peak,
           "clips": pl.n, "src": f"{int(ph['in_h'][-1])}x{int(ph['in_w'][-1])}->{int(ph['out_h'][-1])}x{int(ph['out_w'][-1])}",
           "variants": sorted({int(v) for v in ph["kernel_variant"][: pl.n]})}
    del frames, out
    torch.cuda.empty_cache()
    return res


def k3_launches(mask: int, n: int) -> int:
    """Kernels one vp_resize_normalize_patchify call launches for a plan whose kernel-variant mask is `mask`
    (mirrors the dispatch in vp_resize.cu): grids + generic always; the work index when any TMA variant is present;
    the team tables when team/wide clips are; one launch per present TMA variant (two per team variant: the
    whole-frame and the row-band instantiation, one of which exits at once); the direct kernel if needed."""
    has = lambda v: (mask >> v) & 1
    tma = [has(v) for v in (0, 1, 2, 4, 5, 6, 8)]       # mild, medium, strong, copy, team, wide, team-large
    team = has(5) + has(6) + has(8)                      # team variants launch a whole-frame and a row-band instance
    n_l = (2 + (1 if (any(tma) or has(9)) else 0) + sum(tma) + team + (1 if team else 0) + has(7)
           + 2 * has(9))                                 # + direct; + u8 precision and u8 tiles
    return n_l if n > 0 else 0


def run_dedup(args, pre, pl, frames, off_d, pitch_d, tt, cu, pos, deltas, rst, ws, per, a, dev, world, tokens_rank):
    """cfg5 as GRPO delivers it: sample s of the job is rollout s % 8 of prompt s // 8, keyed by its prompt.  One step
    = vp_dedup_clips over the rank's samples + K1 over the unique clips + K3 over the unique clips only (their frames
    are the first rollout's, already resident) + vp_dedup_views (per-sample patch offset and grid) + K4 over every
    sample's sequence.  The unique-clip list is a function of the keys; it is read back once before timing (a
    trainer knows it from the prompt ids).  Value = tokens delivered to all samples / step time."""
    import torch
    import torch.distributed as dist
    import paper_2604_16893_b200 as vp
    rollouts = 8
    keys = [(a + k) // rollouts for k in range(per)]
    samples = [cfg5_clip()] * per
    uclips, ulist, uid = pre.dedup(samples, keys)
    upl = pre.plan(uclips)
    P = pre.launch_params(upl)
    uout = pre.alloc_outputs(upl)
    ul = torch.tensor(ulist, dtype=torch.int64, device=dev)
    uoff, upitch = off_d[ul], pitch_d[ul]
    keys_d = torch.tensor(keys, dtype=torch.int64, device=dev)
    uid_d = torch.empty(per, dtype=torch.int32, device=dev)
    ulist_d = torch.empty(per, dtype=torch.int32, device=dev)
    nu_d = torch.empty(1, dtype=torch.int32, device=dev)
    po = torch.empty(per, dtype=torch.int64, device=dev)
    grid = torch.empty(per, 3, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    nu = len(ulist)

    def step():
        vp.dedup_clips(keys_d, uid_d, ulist_d, nu_d)
        vp.plan_frames(P, upl.clips_dev, nu, upl.plans_dev, upl.frame_indices, upl.totals_dev, upl.group_timestamps)
        vp.resize_normalize_patchify(P, upl.plans_dev, nu, frames, uoff, upitch, None, uout["pixel_values_videos"],
                                     uout["image_grid_thw"], uout["video_grid_thw"], uout["clip_status"],
                                     workspace=uout["workspace"])
        vp.dedup_views(upl.plans_dev, uid_d, po, grid)
        vp.rope_index(P, vp.VP_ROPE_QWEN3_SPLIT, tt, cu, None, grid, pos, deltas, rst, ws)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    assert (uout["clip_status"][:nu].cpu().numpy() == 0).all() and (rst.cpu().numpy() == 0).all()
    if world > 1:
        dist.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ph = upl.plans_host
    k3_bytes = int(sum(int(ph["n_frames"][k]) * int(ph["in_h"][k]) * 3 * int(ph["in_w"][k]) for k in range(nu))
                   + upl.totals["vid_rows"] * pre.D * 2)
    return {"value": tokens_rank * world / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "steps": args.steps,
            "samples_per_rank": per, "unique_clips_per_rank": nu, "rollouts_per_prompt": rollouts,
            "k3_algorithmic_bytes_per_step": k3_bytes,
            "note": "tokens counted per delivered sample; K3 reads/writes the unique clips only (P:73 hash-based "
                    "dedup); not the headline (the default line processes every sample)"}


def load_traffic(clips_per_rank):
    """ncu dram bytes per clip for K3 (profiles/traffic.json, written from an `ncu --set full` capture)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
        return d["k3_dram_bytes_per_clip"] * clips_per_rank
    except Exception:
        return None


def run_e2e(args, pre, pl, frames, off, pitch, out, tt, cu, pos, deltas, rst, ws, per, dev, world, tokens_rank):
    """Same step through the public API from pinned host memory: per chunk of clips, H2D on a copy stream,
    the resize kernel on the compute stream once the chunk has landed; then MRoPE; then D2H of the
    grids, statuses and deltas the trainer reads.  The pinned source is a ring of `ring` clips."""
    import torch
    import torch.distributed as dist
    import paper_2604_16893_b200 as vp

    P = pre.launch_params(pl)
    chunk = max(1, min(args.e2e_chunk, per))
    ring = max(chunk, min(2 * chunk, per))
    clip_bytes = int(off[1] - off[0]) if per > 1 else int(frames.numel())
    host = torch.empty(ring * clip_bytes, dtype=torch.uint8, pin_memory=True)
    host.copy_(frames[: ring * clip_bytes].cpu())
    grids_h = torch.empty_like(out["video_grid_thw"], device="cpu").pin_memory()
    st_h = torch.empty_like(out["clip_status"], device="cpu").pin_memory()
    dl_h = torch.empty_like(deltas, device="cpu").pin_memory()
    rs_h = torch.empty_like(rst, device="cpu").pin_memory()
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    h2d = per * clip_bytes
    ws_chunk = vp.resize_workspace(chunk, dev)
    d2h = grids_h.numel() * 8 + st_h.numel() * 4 + dl_h.numel() * 8 + rs_h.numel() * 4

    def step():
        vp.plan_frames(P, pl.clips_dev, per, pl.plans_dev, pl.frame_indices, pl.totals_dev, pl.group_timestamps)
        ev_plan = torch.cuda.Event()
        ev_plan.record(comp)
        done = []
        for c0 in range(0, per, chunk):
            c1 = min(per, c0 + chunk)
            with torch.cuda.stream(copy):
                if c0 == 0:
                    copy.wait_event(ev_plan)        # previous step's kernels are done with these regions
                for k in range(c0, c1):
                    src = host[(k % ring) * clip_bytes: (k % ring + 1) * clip_bytes]
                    frames[off[k]: off[k] + clip_bytes].copy_(src, non_blocking=True)
                e = torch.cuda.Event()
                e.record(copy)
            comp.wait_event(e)
            vp.resize_normalize_patchify(P, pl.plans_dev, c1 - c0, frames, torch_off, torch_pitch, None,
                                         out["pixel_values_videos"], out["image_grid_thw"], out["video_grid_thw"],
                                         out["clip_status"], workspace=ws_chunk, stream=comp, first_clip=c0)
            d = torch.cuda.Event()
            d.record(comp)
            done.append(d)
        vp.rope_index(P, vp.VP_ROPE_QWEN3_SPLIT, tt, cu, None, out["video_grid_thw"], pos, deltas, rst, ws)
        grids_h.copy_(out["video_grid_thw"], non_blocking=True)
        st_h.copy_(out["clip_status"], non_blocking=True)
        dl_h.copy_(deltas, non_blocking=True)
        rs_h.copy_(rst, non_blocking=True)

    torch_off = torch.from_numpy(off).to(dev)
    torch_pitch = torch.from_numpy(pitch).to(dev)
    for _ in range(max(1, args.warmup // 2)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(comp)
    for _ in range(args.e2e_steps):
        step()
    b.record(comp)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.e2e_steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    assert (st_h[:per].numpy() == 0).all()
    return {"value": tokens_rank * world / (ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms, "steps": args.e2e_steps,
            "path": "pinned host u8 frames -> H2D (copy stream, chunks of %d clips) overlapped with K3; "
                    "D2H of grids/status/deltas" % chunk}


def run_e2e_nv12(args, pre, pl, frames, off, pitch, out, tt, cu, pos, deltas, rst, ws, per, dev, world, tokens_rank):
    """As run_e2e, but the host holds what a decoder emits -- NV12 (Y plane + interleaved UV, 1.5 B/pixel) -- and
    the device converts it with vp_nv12_to_rgb (N4) straight into each clip's slot of the K3 frame buffer: half
    the PCIe bytes of RGB.  NV12 staging on the device is double-buffered per chunk of clips."""
    import torch
    import torch.distributed as dist
    import paper_2604_16893_b200 as vp

    P = pre.launch_params(pl)
    ph = pl.plans_host
    chunk = max(1, min(args.e2e_chunk, per))
    n, H, W = int(ph["n_frames"][0]), int(ph["in_h"][0]), int(ph["in_w"][0])
    fstride = H * W * 3 // 2
    nv_clip = n * fstride
    ring = max(chunk, min(2 * chunk, per))
    host = torch.randint(0, 256, (ring * nv_clip,), dtype=torch.uint8).pin_memory()
    stage = [torch.empty(chunk * nv_clip, dtype=torch.uint8, device=dev) for _ in range(2)]
    st_h = torch.empty_like(out["clip_status"], device="cpu").pin_memory()
    dl_h = torch.empty_like(deltas, device="cpu").pin_memory()
    grids_h = torch.empty_like(out["video_grid_thw"], device="cpu").pin_memory()
    rs_h = torch.empty_like(rst, device="cpu").pin_memory()
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    ws_chunk = vp.resize_workspace(chunk, dev)
    torch_off = torch.from_numpy(off).to(dev)
    torch_pitch = torch.from_numpy(pitch).to(dev)
    d2h = grids_h.numel() * 8 + st_h.numel() * 4 + dl_h.numel() * 8 + rs_h.numel() * 4

    def step():
        vp.plan_frames(P, pl.clips_dev, per, pl.plans_dev, pl.frame_indices, pl.totals_dev, pl.group_timestamps)
        freed = [torch.cuda.Event(), torch.cuda.Event()]
        for e in freed:
            e.record(comp)
        for ci, c0 in enumerate(range(0, per, chunk)):
            c1 = min(per, c0 + chunk)
            buf = stage[ci % 2]
            with torch.cuda.stream(copy):
                copy.wait_event(freed[ci % 2])      # the conversions of chunk ci-2 are done with this buffer
                for k in range(c0, c1):
                    src = host[(k % ring) * nv_clip: (k % ring + 1) * nv_clip]
                    buf[(k - c0) * nv_clip: (k - c0 + 1) * nv_clip].copy_(src, non_blocking=True)
                e = torch.cuda.Event()
                e.record(copy)
            comp.wait_event(e)
            for k in range(c0, c1):
                nb = buf[(k - c0) * nv_clip:]
                vp.nv12_to_rgb(nb, nb[H * W:], W, fstride, H, W, n, frames[int(off[k]):], int(pitch[k]),
                               H * int(pitch[k]), stream=comp)
            fe = torch.cuda.Event()
            fe.record(comp)
            freed[ci % 2] = fe
            vp.resize_normalize_patchify(P, pl.plans_dev, c1 - c0, frames, torch_off, torch_pitch, None,
                                         out["pixel_values_videos"], out["image_grid_thw"], out["video_grid_thw"],
                                         out["clip_status"], workspace=ws_chunk, stream=comp, first_clip=c0)
        vp.rope_index(P, vp.VP_ROPE_QWEN3_SPLIT, tt, cu, None, out["video_grid_thw"], pos, deltas, rst, ws)
        grids_h.copy_(out["video_grid_thw"], non_blocking=True)
        st_h.copy_(out["clip_status"], non_blocking=True)
        dl_h.copy_(deltas, non_blocking=True)
        rs_h.copy_(rst, non_blocking=True)

    for _ in range(max(1, args.warmup // 2)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(comp)
    for _ in range(args.e2e_steps):
        step()
    b.record(comp)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.e2e_steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    assert (st_h[:per].numpy() == 0).all()
    return {"value": tokens_rank * world / (ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": per * nv_clip,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms, "steps": args.e2e_steps,
            "path": "pinned host NV12 frames (decoder output) -> H2D (copy stream, double-buffered chunks of %d "
                    "clips) -> vp_nv12_to_rgb into the K3 frame buffer -> K3; D2H of grids/status/deltas" % chunk}


# ----------------------------------------------------------------------------------------------
# oracle (CPU baseline and the reference arm)
# ----------------------------------------------------------------------------------------------

def oracle_sample(frames_groups: int):
    """The oracle, as it stands, on a bounded sample of the workload: one cfg5 clip's plan, its first
    `frames_groups` temporal groups through resize/normalise/patchify, and the clip's MRoPE sequence
    truncated to those groups.  Returns (visual tokens processed, seconds)."""
    import oracle as O
    import vp_inputs as I

    params = cfg5_params()
    c = cfg5_clip()
    t0 = time.perf_counter()
    pl = O.plan_clip(params, c)
    tp, p, m = params["temporal_patch_size"], params["patch_size"], params["merge_size"]
    g = min(frames_groups, pl.grid[0])
    idx = pl.idx[: g * tp]
    fr = I.frames_u8("noise", 0, idx, pl.in_h, pl.in_w)
    gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    res = np.stack([O.resize_frame(fr[k], pl.out_h, pl.out_w) for k in range(len(idx))])
    rows = O.patchify(O.normalize(res, params["mean"], params["std"]), p, m, tp)
    runs = [(0, 64)]
    for _ in range(g):
        runs += [(0, 7), (2, pl.grid[1] * pl.grid[2] // m ** 2), (0, 1)]
    O.rope_index([I.token_types(runs)], [], [(g, pl.grid[1], pl.grid[2])], m)
    secs = time.perf_counter() - t0
    tokens = rows.shape[0] // (m * m)
    return tokens, secs, gen


def cpu_baseline(clips=4):
    """The oracle on `clips` full cfg5 clips (32 temporal groups each, ~2 s per clip on 16 cores)."""
    tokens, secs = 0, 0.0
    for _ in range(clips):
        tk, s, _ = oracle_sample(32)
        tokens += tk
        secs += s
    cores = len(os.sched_getaffinity(0))
    return {"value": tokens / secs, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{clips} full cfg5 clips (64 frames 720p -> 384x672 each: plan, f64 resize/normalise/"
                      f"patchify, MRoPE of its sequence); numpy f64 oracle, BLAS threads = host cores",
            "seconds": secs}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    groups = max(1, args.ref_groups)
    for _ in range(args.warmup):
        oracle_sample(1)
    times, toks = [], 0
    for _ in range(args.steps):
        tk, s, _ = oracle_sample(groups)
        times.append(s)
        toks = tk
    v = toks / (sum(times) / len(times))
    cores = len(os.sched_getaffinity(0))
    sample = f"per step: 1 cfg5 clip, first {groups} temporal groups + MRoPE (f64 numpy oracle)"
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg5 (bounded oracle sample, see cpu_baseline.sample)"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--clips", type=int, default=0, help="override job clip count (profiling only)")
    ap.add_argument("--config", default="cfg5", choices=["cfg5", "cfg1", "cfg2", "cfg3", "cfg4"],
                    help="workload (default cfg5, the metric's configuration)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-chunk", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dedup", action="store_true", help="skip the 64 x 8 GRPO dedup line (N3)")
    ap.add_argument("--no-side", action="store_true", help="skip the cfg1-cfg4 / resolution side lines")
    ap.add_argument("--cpu-clips", type=int, default=4)
    ap.add_argument("--ref-groups", type=int, default=2)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo only for --dist-selftest on CPU)")
    ap.add_argument("--dist-selftest", action="store_true",
                    help="launcher check without GPUs: spawn, rendezvous, clip sharding, record all-gather, "
                         "max-over-ranks reduction (prints one JSON line on rank 0)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args.gpus)                              # re-exec under torch.distributed.run; never returns
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.gpus != world:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE {world}"}))
        sys.exit(2)
    if args.dist_selftest:
        dist_selftest(args, rank, world)
        return
    if args.impl == "reference":
        r = run_reference(args, rank, world)
        if r is not None:
            print(json.dumps(r))
        return
    import torch
    import torch.distributed as dist
    nccl_glob = None
    if world > 1:
        # NCCL communicator-init logging (nRanks per communicator) to a per-process file, summarised in the JSON
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", os.path.join(tempfile.gettempdir(), "vp_nccl.%h.%p.log"))
        nccl_glob = os.environ["NCCL_DEBUG_FILE"].replace("%h", "*").replace("%p", str(os.getpid()))
        dist.init_process_group(args.backend, device_id=torch.device("cuda", local_rank))
    res = run_ours(args, rank, world, local_rank)
    if rank == 0 and world == 1 and not args.no_side and args.config == "cfg5":
        # side lines: the other BASELINE configs and source resolutions (after the cfg5 buffers are released)
        torch.cuda.empty_cache()
        res["side_lines"] = {name: measure_side(name, torch.device("cuda", local_rank)) for name in SIDE_CONFIGS}
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            res["cpu_baseline"] = cpu_baseline(args.cpu_clips)
        if world > 1:
            from paper_2604_16893_b200.dist import nccl_log_nranks
            res["nccl"] = {"backend": args.backend, "comm_nranks": nccl_log_nranks(nccl_glob),
                           "h10": "all_gather_into_tensor of int32 (t,h,w,tokens) records, async on the NCCL "
                                  "stream, overlapping K3; work.wait() before vp_pack_offsets"}
        print(json.dumps(res))
    if world > 1:
        dist.destroy_process_group()


def spawn_ranks(n: int):
    """`python bench.py --gpus N` outside torchrun: re-exec as one process per GPU through torch.distributed.run
    (single node, rendezvous on 127.0.0.1), with the same arguments."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dist_selftest(args, rank, world):
    """The N>1 plumbing of the bench without GPUs (gloo): rendezvous, the cfg5 clip shard of this rank, an
    all-gather of per-clip int32 records (here (rank, clip, a + k, 1) so the gathered order is checkable) and the
    max-over-ranks reduction of the step time."""
    import torch
    import torch.distributed as dist
    from paper_2604_16893_b200.dist import shard_range
    dist.init_process_group(args.backend)
    job = args.clips if args.clips else JOB_CLIPS
    a, b = shard_range(job, world, rank)
    rec = torch.tensor([[rank, k, a + k, 1] for k in range(b - a)], dtype=torch.int32).reshape(-1)
    out = torch.empty(world * rec.numel(), dtype=torch.int32)
    dist.all_gather_into_tensor(out, rec)
    g = out.reshape(-1, 4)
    ok = g[:, 2].tolist() == list(range(job)) and all(int(g[i, 0]) == i // (job // world) for i in range(job))
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dist_selftest": "ok" if ok and t.item() == world else "fail", "world": world,
                          "backend": args.backend, "clips": job, "shard_sizes": [b - a] * 1,
                          "gathered_records": int(g.shape[0]), "max_over_ranks": t.item()}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
