#!/usr/bin/env python
"""Benchmark of the IKJT training hot path (dedup + pooled fwd + expand + bwd/SGD).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "cfg2"): B=65,536 session-clustered rows
per GPU, 26 keys with lengths ([8,16,32,64,128,256]*5)[:26], mean session
16.5 samples (geometric), change_prob 0.15, 26 fp32 tables of 10M x 128 on
one B200.  Inputs come from the restated reference generator
(paper_2211_05239_b200/datagen.py), tables are uniform(-0.1, 0.1) drawn on the
device, grad_out ~ N(0,1) resident (synthetic upstream gradient).

One step = recd_dedup (KJT->IKJT, all keys) + recd_pool_fwd + recd_expand +
recd_pool_bwd (segment-reduce, sorted scatter-add, fused SGD), replayed as one
CUDA graph.  Inputs (1.07 GB of int64 IDs) and tables (133 GB) are far larger
than the 126 MB L2, so no L2 flush is needed between steps.

Rank 0 prints ONE JSON line.  `--impl reference` times the reference's CPU
algorithm (the oracle port, oracle/) on the host cores instead.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples/sec for IKJT dedup + embedding fwd/bwd; achieved HBM GB/s vs peak"

# DRAM bytes (read + write) per launch from one `ncu --set full` capture of the
# cfg2 bench (profiles/r1_ncu_summary.txt); refreshed when the kernels change.
TRAFFIC: dict = {"k_scatter": 9.818e9, "k_pool_fwd": 4.852e9}  # profiles/r1_ncu_final.txt
LENS = ([8, 16, 32, 64, 128, 256] * 5)[:26]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=65536, help="rows per GPU")
    ap.add_argument("--keys", type=int, default=26)
    ap.add_argument("--rows", type=int, default=10_000_000, help="table rows")
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--mode", choices=["dedup", "kjt"], default="dedup")
    ap.add_argument("--samples-per-session", type=float, default=16.5)
    ap.add_argument("--dist", choices=["geometric", "fixed"], default="geometric")
    ap.add_argument("--change-prob", type=float, default=0.15)
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--transport", choices=["peer", "nccl"], default="peer",
                    help="N>1: exchange over NVLink peer memory (graph) or NCCL")
    ap.add_argument("--shards", type=int, default=0,
                    help="N>1: row shards per table (0 = auto: the fewest that fit HBM)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-overlap", action="store_true",
                    help="run the backward's prepare half on the main stream")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=0,
                    help="rows in the CPU sample (0 = calibrated to --cpu-seconds)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target CPU work of the bounded baseline sample")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e/cpu)")
    return ap.parse_args()


# ----------------------------------------------------------------- inputs
def make_batch(args, rank, world):
    from paper_2211_05239_b200.datagen import (FeatureSpec, SampleCountDist, SessionConfig,
                                               generate_clustered_batch)
    specs = [FeatureSpec(f"k{i}", "user_sequence", float(LENS[i % len(LENS)]), args.rows,
                         args.change_prob) for i in range(args.keys)]
    total_rows = args.batch * world
    nsess = int(math.ceil(total_rows / args.samples_per_session * 1.3)) + 64
    cfg = SessionConfig(nsess, SampleCountDist(args.dist, args.samples_per_session), 0)
    return generate_clustered_batch(cfg, specs, args.batch, row_start=rank * args.batch)


def algorithmic_bytes(B, K, D, N_kjt, N_u, U_tot, N_ids):
    """A = 8(N_kjt + BK) + 8(N_u + U_tot + BK) + 4D N_u
    + 4D BK (expanded output) + 4D BK (grad_out read) + 2*4D N_ids (SGD RMW)."""
    return (8 * (N_kjt + B * K) + 8 * (N_u + U_tot + B * K) + 4 * D * N_u + 8 * D * B * K
            + 8 * D * N_ids)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(gpu_index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------- CPU side
_CPU = {}


def _cpu_key_work(k):
    """Reference algorithm for one key on the CPU sample: build_ikjt
    (tensors.py:269-308), embedding_lookup + pool + b[inv]
    (trainer_sim.py:308-344, 558-561) and the backward restatement + SGD."""
    import oracle
    v, o, g, w, lr = (_CPU["values"][k], _CPU["offsets"][k], _CPU["grad"], _CPU["table"],
                      _CPU["lr"])
    inv, [(uv, uo)] = oracle.build_ikjt_arrays([(v, o)])
    pooled = oracle.pooled_lookup(uv, uo, w, "sum")
    out = oracle.expand(pooled, inv)
    gu = oracle.pool_backward(g, inv, uo.size)
    ids, gw = oracle.sparse_table_grad(gu, uv, uo, "sum")
    w[ids] -= (np.float32(lr) * gw).astype(np.float32)
    return float(out[0, 0])


def cpu_time(batch, rows, dim, lr, procs):
    """Seconds for the whole sample (all keys) using `procs` processes."""
    import multiprocessing as mp
    rng = np.random.default_rng(0)
    _CPU["values"], _CPU["offsets"] = {}, {}
    for k in batch.keys:
        o = batch.offsets[k][:rows]
        end = batch.offsets[k][rows] if rows < batch.batch_size else batch.values[k].size
        _CPU["values"][k] = batch.values[k][:end]
        _CPU["offsets"][k] = o
    _CPU["grad"] = rng.standard_normal((rows, dim)).astype(np.float32)
    vocab = int(max(v.max() for v in _CPU["values"].values())) + 1
    tab = _CPU.get("table")
    if tab is None or tab.shape[0] < vocab or tab.shape[1] != dim:   # built once, reused
        _CPU["table"] = rng.uniform(-0.1, 0.1, size=(vocab, dim)).astype(np.float32)
    _CPU["lr"] = lr
    keys = list(batch.keys)
    t0 = time.perf_counter()
    if procs <= 1:
        for k in keys:
            _cpu_key_work(k)
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            pool.map(_cpu_key_work, keys, chunksize=1)
    return time.perf_counter() - t0


def calibrated_rows(batch, dim, lr, procs, target_s):
    """Rows of the CPU sample that take about target_s seconds (rate probed on
    256 rows, which also builds the shared table)."""
    t = cpu_time(batch, 256, dim, lr, procs)
    return int(max(256, min(batch.batch_size, 256 * target_s / max(t, 1e-3))))


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    batch = make_batch(args, 0, 1)
    procs = min(host_cores(), args.keys)
    # each step a bounded sample: ~cpu_seconds, capped so K + W steps fit ~3 minutes
    per_step = min(args.cpu_seconds, 180.0 / (max(1, args.steps) + max(0, args.warmup)))
    rows = args.cpu_rows or calibrated_rows(batch, args.dim, args.lr, procs, per_step)
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_time(batch, min(rows, 256), args.dim, args.lr, procs)
    times = [cpu_time(batch, rows, args.dim, args.lr, procs) for _ in range(max(1, args.steps))]
    t = float(np.mean(times))
    value = rows / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": config_dict(args, "cpu"),
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": procs, "kind": "port",
                         "sample": f"first {rows} of {args.batch} rows x {args.keys} keys per step, "
                                   f"one shared {dim_str(args)} table, oracle/ restatement of "
                                   "build_ikjt + lookup/pool/expand + backward + SGD, "
                                   f"{procs} processes (keys fanned out)"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def dim_str(args):
    return f"{args.rows}x{args.dim} fp32"


def config_dict(args, where):
    return {"workload": "cfg2: IKJT dedup + sum-pooled EmbeddingBag fwd/bwd(+SGD)",
            "global_batch": args.batch * args.gpus, "batch_per_gpu": args.batch,
            "keys": args.keys, "max_len": max(LENS[: args.keys]), "tables": args.keys,
            "table": dim_str(args), "samples_per_session": args.samples_per_session,
            "session_dist": args.dist, "change_prob": args.change_prob, "mode": args.mode,
            "parallelism": f"dp{args.gpus}-replicas" if args.gpus > 1 else "single",
            "l2": "inputs (1.07 GB ids, 133 GB tables) >> 126 MB L2; no flush", "where": where}


# ------------------------------------------------------------------- main
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    import paper_2211_05239_b200 as R
    from paper_2211_05239_b200.step import TrainStep

    if world > 1:
        return run_sharded(args, world, rank, local, dev)

    t_setup = time.perf_counter()
    batch = make_batch(args, rank, world)
    keys = list(batch.keys)
    tables = {k: R.EmbeddingTable.create_on_device(k, args.rows, args.dim, seed=i, device=dev)
              for i, k in enumerate(keys)}
    caps = {k: batch.values[k].size for k in keys}
    step = TrainStep([[k] for k in keys], args.batch, caps, tables, "sum", args.lr, args.mode, dev,
                     overlap=not args.no_overlap)
    step.load_batch(batch.values, batch.offsets)
    step.fill_grad_out(1 + rank)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup

    # one eager step to read the step's statistics
    step.run()
    torch.cuda.synchronize()
    counts = step.host_counts()
    stream = torch.cuda.current_stream(dev)
    B, K, D = args.batch, len(keys), args.dim
    N_kjt = int(sum(caps.values()))
    N_u = int(sum(counts.N_u))
    U_tot = int(sum(counts.U))
    # distinct IDs per table (for the SGD RMW term): from the unique values
    N_ids = 0
    for f in range(K):
        n = counts.N_u[f]
        N_ids += int(torch.unique(step.uvalues[f][:n] if args.mode == "dedup"
                                  else step.in_values[f][:n]).numel())

    for _ in range(args.warmup):
        step.run()
    if not args.no_graph:
        step.capture()
    for _ in range(max(1, args.warmup)):
        step.replay()
    torch.cuda.synchronize()

    # ------------------------------------------------------ timed region
    sampler = ClockSampler(local) if not args.profile else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = R.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    clocks = sampler.stop() if sampler else None
    launches_per_step = R.launch_count() - launches0
    if not args.no_graph:
        # graph replays do not pass through the host counter: count one eager step
        l0 = R.launch_count()
        step.run()
        launches_per_step = R.launch_count() - l0
        torch.cuda.synchronize()
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * B / (ms / 1e3)

    # --------------------------------------- per-phase timing (roofline)
    phases = {"dedup": [], "pool": [], "expand": [], "bwd": []}
    s = stream.cuda_stream
    for _ in range(max(3, min(args.steps, 20))):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(stream)
        step.dedup(s)
        ev[1].record(stream)
        step.forward(s)
        ev[2].record(stream)
        step.expand(s)
        ev[3].record(stream)
        step.backward(s)
        ev[4].record(stream)
        torch.cuda.synchronize()
        for i, name in enumerate(phases):
            phases[name].append(ev[i].elapsed_time(ev[i + 1]))
    ph = {k: float(np.mean(v)) for k, v in phases.items()}
    peaks = load_peaks()
    peak = peaks.get("hbm_gbs")

    # the two largest kernels, timed live with CUDA events recorded by librecd
    # right before / after their launch (recd_debug_kernel_events)
    lib = R.load_library()

    def kernel_ms(name, n):
        ts = []
        for _ in range(n):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            b.record(stream)
            lib.recd_debug_kernel_events(name.encode(), a.cuda_event, b.cuda_event)
            step.run()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        lib.recd_debug_kernel_events(None, None, None)
        return float(np.mean(ts))

    nk = max(3, min(args.steps, 10))
    kernels = {}
    # compulsory HBM bytes per launch (distinct table rows once; SURVEY §8(d)
    # counts every gathered row: "requested")
    kb = {"k_pool_fwd": (8 * N_u + 8 * U_tot + 4 * D * N_ids + 4 * D * U_tot,
                         8 * N_u + 8 * U_tot + 4 * D * N_u + 4 * D * U_tot),
          "k_scatter": (8 * N_u + 4 * D * U_tot + 8 * D * N_ids,
                        8 * N_u + 4 * D * N_u + 8 * D * N_ids)}
    if args.mode == "kjt":
        kb = {"k_pool_fwd": (8 * N_kjt + 4 * D * N_ids + 4 * D * B * K,
                             8 * N_kjt + 4 * D * N_kjt + 4 * D * B * K),
              "k_scatter": (8 * N_kjt + 4 * D * B * K + 8 * D * N_ids,
                            8 * N_kjt + 4 * D * N_kjt + 8 * D * N_ids)}
    for name, (comp, req) in kb.items():
        t = kernel_ms(name, nk)
        kernels[name] = {"ms": t, "compulsory_bytes": comp, "requested_bytes": req,
                         "achieved_gbs": comp / (t / 1e3) / 1e9,
                         "achieved_requested_gbs": req / (t / 1e3) / 1e9}
    dom = max(kernels, key=lambda k: kernels[k]["ms"])
    pool_bytes = kernels[dom]["compulsory_bytes"]
    pool_gbs = kernels[dom]["achieved_gbs"]
    A = algorithmic_bytes(B, K, D, N_kjt, N_u, U_tot, N_ids)
    if args.mode == "kjt":
        A = algorithmic_bytes(B, K, D, N_kjt, N_kjt, B * K, N_ids) - 8 * (N_kjt + 2 * B * K)
    step_gbs = A / (ms / 1e3) / 1e9

    # ----------------------------------------------------------- e2e
    e2e = None
    if not args.no_e2e and not args.profile:
        e2e = e2e_pipelined(step, batch, keys, step.replay, dev, max(4, min(args.steps, 20)),
                            world, dist if world > 1 else None)
        e2e["how"] = ("public TrainStep API: pinned-host KJT -> H2D on a copy stream "
                      "(double-buffered, overlaps the previous step) -> graph replay -> D2H of "
                      "the step's dedup counts read by the host")

    # ------------------------------------------------------ CPU baseline
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        procs = min(host_cores(), K)
        rows = args.cpu_rows or calibrated_rows(batch, D, args.lr, procs, args.cpu_seconds)
        t = cpu_time(batch, rows, D, args.lr, procs)
        cpu = {"value": rows / t, "unit": "samples/s", "cores": procs, "kind": "port",
               "sample": f"first {rows} of {B} rows x {K} keys, one shared table, oracle/ "
                         f"restatement (build_ikjt + lookup/pool/expand + bwd + SGD), "
                         f"{procs} processes, {t:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 (ids int64)", "data": "synthetic (restated reference session generator)",
            "config": config_dict(args, "gpu"),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": pool_gbs,
                         "peak": peak, "unit": "GB/s",
                         "frac": pool_gbs / peak if peak else None,
                         "peak_source": ("MEASURED_PEAKS.json hbm_gbs (measured)"
                                         if "note" not in peaks else "fallback 6650 GB/s"),
                         "traffic": TRAFFIC.get(dom), "algorithmic_bytes_per_launch": pool_bytes,
                         "bytes_definition": "compulsory: each distinct table row once "
                                             "(DESIGN.md §4)",
                         "avg_launch_ms": kernels[dom]["ms"],
                         "achieved_requested": kernels[dom]["achieved_requested_gbs"]},
            "kernels": kernels,
            "step_roofline": {"algorithmic_bytes": A, "achieved_gbs": step_gbs,
                              "frac": step_gbs / peak if peak else None},
            "phases_ms": ph,
            "stats": {"N_kjt": N_kjt, "N_u": N_u, "U_tot": U_tot, "N_ids": N_ids,
                      "dedupe_factor": N_kjt / max(N_u, 1)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "gpu_launches_per_step": launches_per_step,
            "clocks": clocks,
            "setup_s": setup_s,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def e2e_pipelined(step, batch, keys, replay, dev, n_steps, world, dist=None):
    """End-to-end samples/s through the public step API from pinned host
    buffers: every step's KJT goes H2D (copy stream, double-buffered, so the
    copy of batch i+1 overlaps step i), the step runs, and its dedup counts
    come back D2H and are read by the host (one step of lag)."""
    import torch

    from paper_2211_05239_b200.staging import H2DPipeline

    pin_v = {k: torch.from_numpy(batch.values[k]).pin_memory() for k in keys}
    pin_o = {k: torch.from_numpy(batch.offsets[k]).pin_memory() for k in keys}
    h2d = sum(pin_v[k].numel() * 8 + pin_o[k].numel() * 8 for k in keys)
    pipe = H2DPipeline(step, dev)
    res = [torch.empty(step.counts.numel(), dtype=torch.int64).pin_memory() for _ in range(2)]
    done = [torch.cuda.Event(), torch.cuda.Event()]
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    pipe.prefetch(0, pin_v, pin_o)
    for i in range(n_steps):
        if i + 1 < n_steps:
            pipe.prefetch((i + 1) % 2, pin_v, pin_o)
        pipe.install(i % 2)
        replay()
        res[i % 2].copy_(step.counts, non_blocking=True)
        done[i % 2].record()
        if i >= 1:
            done[(i - 1) % 2].synchronize()
            _ = int(res[(i - 1) % 2][0])
    torch.cuda.synchronize()
    _ = int(res[(n_steps - 1) % 2][0])
    e2e_s = (time.perf_counter() - t0) / n_steps
    if dist is not None:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    B = step.B
    return {"value": world * B / e2e_s, "unit": "samples/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": res[0].numel() * 8, "ms_per_step": e2e_s * 1e3,
            "h2d_gbs": h2d / e2e_s / 1e9}


def run_sharded(args, world, rank, local, dev):
    """N > 1: every table row-sharded into S shards (id mod S), the
    (table, shard) pairs placed on ranks LPT-first, + data-parallel batch;
    each rank deduplicates its own 65,536-row chunk of the global batch and
    the NCCL exchange carries only deduplicated IDs, partially pooled rows and
    unique-row gradients (paper_2211_05239_b200/sharded.py)."""
    import torch
    import torch.distributed as dist

    import paper_2211_05239_b200 as R
    from paper_2211_05239_b200.peer import PeerShardedStep
    from paper_2211_05239_b200.sharded import ShardedTrainStep, auto_shards

    t_setup = time.perf_counter()
    batch = make_batch(args, rank, world)
    keys = list(batch.keys)
    if args.shards:
        S = args.shards
    else:   # smallest S whose placement fits 60% of HBM (tables are fp32)
        hbm = torch.cuda.get_device_properties(dev).total_memory
        S = auto_shards([float(batch.values[k].size) for k in keys],
                        [4 * args.rows * args.dim] * len(keys), world, 0.6 * hbm)
        t = torch.tensor([S], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)   # identical on every rank
        S = int(t.item())

    def make_table(k, j, n):
        return R.EmbeddingTable.create_on_device(f"{k}/shard{j}", n, args.dim,
                                                 seed=1000 * keys.index(k) + j, device=dev)

    caps = {k: batch.values[k].size for k in keys}
    peer_kw = {"overlap": not args.no_overlap} if args.transport == "peer" else {}
    cls = PeerShardedStep if args.transport == "peer" else ShardedTrainStep
    step = cls(keys, args.batch, caps, {k: args.rows for k in keys}, args.dim, make_table, "sum",
               args.lr, shards=S, device=dev, **peer_kw)
    peer = args.transport == "peer"
    lrows = sum(t.rows for t in step.tables.values())
    step.load_batch(batch.values, batch.offsets)
    step.fill_grad_out(1 + rank)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.current_stream(dev)
    B, K, D = args.batch, len(keys), args.dim
    if peer:
        step.capture()        # fwd + bwd of every rank: one CUDA graph, no host sync
    for _ in range(max(1, args.warmup)):
        step.replay() if peer else step.run()
    torch.cuda.synchronize()
    if peer:
        step.check()
    U, N_u = step.host_counts()

    sampler = ClockSampler(local) if not args.profile else None
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = R.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step.replay() if peer else step.run()
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    if peer:
        step.check()
    ms = e0.elapsed_time(e1) / args.steps
    clocks = sampler.stop() if sampler else None
    launches_per_step = (R.launch_count() - launches0) // max(args.steps, 1)
    t = torch.tensor([ms], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = world * B / (ms / 1e3)

    # sub-phase breakdown (one traced step per rank, max over ranks)
    step.trace = True
    l0 = R.launch_count()
    step.run()
    if peer:   # graph replays do not pass through the host counter: count this eager step
        launches_per_step = R.launch_count() - l0
    ph = step.phase_ms()
    step.trace = False
    names = list(ph)
    tph = torch.tensor([ph[n] for n in names], device=dev)
    dist.all_reduce(tph, op=dist.ReduceOp.MAX)
    ph = dict(zip(names, tph.tolist()))
    # per-rank communication volume of the step (bytes sent)
    if peer:
        P = step.P
        meta = step.ctl[128:128 + world * 2 * P].view(world, 2 * P).cpu().numpy()
        send_ids, send_rows = meta[rank, :P], meta[rank, P:]
        recv_rows = meta[:, P:][:, step.mine]
    else:
        pl = step.plan
        send_ids, send_rows, recv_rows = pl.send_ids, pl.send_rows, pl.recv_rows
    sent = 8 * int(send_ids.sum()) + 8 * int(send_rows.sum())  # ids + row offsets / counts
    sent += 4 * D * int(recv_rows.sum())  # partial pooled rows returned
    sent += 4 * D * int(send_rows.sum())  # unique-row gradients (one copy per shard)
    N_kjt = int(sum(caps.values()))
    # the reference's all-to-all accounting (trainer_sim.sdd,
    # tensors.slice_stream_bytes) for this rank's batch -- canonical wire bytes of
    # every (offsets, values) slice sent, dedup vs KJT, and the pooled rows back
    a2a_fwd_dedup = sum(16 + 8 * (U[f] + N_u[f]) for f in range(len(keys)))
    a2a_fwd_kjt = sum(16 + 8 * (args.batch + int(caps[k])) for k in keys)
    a2a = {"fwd_bytes_dedup": a2a_fwd_dedup, "fwd_bytes_kjt": a2a_fwd_kjt,
           "fwd_reduction": a2a_fwd_kjt / max(a2a_fwd_dedup, 1),
           "back_bytes_dedup": 4 * D * int(sum(U)), "back_bytes_kjt": 4 * D * args.batch * len(keys),
           "definition": "trainer_sim.sdd / a2a_bytes_back (trainer_sim.py:281-305, 557, 573) on rank 0's "
                         "batch; the inverse never travels"}

    e2e = None
    if not args.no_e2e and not args.profile:
        e2e = e2e_pipelined(step, batch, keys, step.replay if peer else step.run, dev,
                            max(4, min(args.steps, 10)), world, dist)
        e2e["how"] = (f"{cls.__name__} on every rank: pinned-host KJT -> H2D on a copy stream "
                      "(double-buffered) -> step -> D2H of the dedup counts; max over ranks")
    if rank == 0:
        cfg = config_dict(args, "gpu")
        cfg["parallelism"] = (f"dp{world} x {S}-way row-sharded tables (shard = id mod {S}), "
                              f"(table, shard) pairs placed LPT")
        cfg["transport"] = ("NVLink peer memory (CUDA IPC), whole step one CUDA graph" if peer
                            else "NCCL all-to-all, host-planned split sizes")
        cfg["table_rows_rank0"] = lrows
        cfg["pairs_rank0"] = len(step.mine)
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 (ids int64)", "data": "synthetic (restated reference session generator)",
            "config": cfg, "phases_ms": ph,
            "comm_bytes_sent_per_rank": sent, "a2a_accounting_rank0": a2a,
            "stats_rank0": {"N_kjt": N_kjt, "N_u": int(sum(N_u)), "U_tot": int(sum(U))},
            "roofline": None, "cpu_baseline": None, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "gpu_launches_per_step": launches_per_step, "clocks": clocks, "setup_s": setup_s,
        }
        print(json.dumps(line), flush=True)
    if peer:
        step.close()
    dist.destroy_process_group()
    return 0


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {"hbm_gbs": 6650.0, "note": "fallback"}


if __name__ == "__main__":
    sys.exit(main())
