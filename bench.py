#!/usr/bin/env python
"""Benchmark of the IKJT training hot path (dedup + pooled fwd + expand + bwd/SGD).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2|cfg1]

Workload (BASELINE.json configs[1], "cfg2", the default): B=65,536
session-clustered rows per GPU, 26 keys with lengths
([8,16,32,64,128,256]*5)[:26], mean session 16.5 samples (geometric),
change_prob 0.15, 26 fp32 tables of 10M x 128 on one B200.  `--config cfg1`
is BASELINE.json configs[0]: B=4096, 8 keys of lengths 4..32, one shared
1M x 64 table.  Inputs come from the restated reference generator
(tools/datagen.py), tables are uniform(-0.1, 0.1) drawn on the device,
grad_out ~ N(0,1) resident (synthetic upstream gradient).

One step = recd_dedup (KJT->IKJT, all keys) + recd_pool_fwd + recd_expand +
recd_pool_bwd (segment-reduce, sorted scatter-add, fused SGD), replayed as one
CUDA graph.  cfg2's inputs (1.07 GB of int64 IDs) and tables (133 GB) are far
larger than the 126 MB L2, so no L2 flush is needed between steps; cfg1 fits
in L2 and says so in its config.

N > 1: `--gpus N` launches N ranks itself (torch.distributed.run, one process
per GPU, NCCL) unless it already runs under a launcher (WORLD_SIZE set, which
must equal N).  Every rank deduplicates its own 65,536 rows; tables are
row-sharded over the ranks (peer.PeerShardedStep).  Timing is the max over
ranks of CUDA-event time; rank 0 prints ONE JSON line.

`--impl reference` times the reference's own CPU implementation: the
unmodified `sessiondedup` package installed at baseline/_ref (build_ikjt,
embedding_lookup, pool, the b[inv] expansion), plus the backward restatement
of oracle/ (the reference has no backward); the oracle port
stands in only if baseline/_ref is absent.  Rows are fanned out over all host
cores in split_batch chunks (trainer_sim.py:416-446) by a persistent process
pool; a 1-core figure is reported beside it.
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

CONFIGS = {
    "cfg2": {"batch": 65536, "lens": ([8, 16, 32, 64, 128, 256] * 5)[:26], "rows": 10_000_000,
             "dim": 128, "shared_table": False, "sessions": None,
             "workload": "cfg2: IKJT dedup + sum-pooled EmbeddingBag fwd/bwd(+SGD), 26 keys x "
                         "10M x 128 tables",
             "l2": "inputs (1.07 GB ids, 133 GB tables) >> 126 MB L2; no flush"},
    "cfg1": {"batch": 4096, "lens": [4, 8, 12, 16, 20, 24, 28, 32], "rows": 1_000_000, "dim": 64,
             "shared_table": True, "sessions": 600,
             "workload": "cfg1: IKJT dedup + sum-pooled EmbeddingBag fwd/bwd(+SGD), 8 keys, one "
                         "shared 1M x 64 table",
             "l2": "touched data (~60 MB/step) fits in the 126 MB L2: launch-bound, no flush"},
}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg2")
    ap.add_argument("--batch", type=int, default=0, help="rows per GPU (0 = the config's)")
    ap.add_argument("--keys", type=int, default=0, help="0 = the config's")
    ap.add_argument("--rows", type=int, default=0, help="table rows (0 = the config's)")
    ap.add_argument("--dim", type=int, default=0)
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
    ap.add_argument("--pipeline", action="store_true",
                    help="N=1: cross-step pipelining (the next batch's dedup + backward prepare "
                         "on a side stream during the current step; A/B: 4.86 vs 4.89 ms, e2e lower)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-raw-share", type=float, default=None,
                    help="row-coded e2e: share of the IDs copied raw (default: the balance model)")
    ap.add_argument("--e2e-wire", choices=["auto", "rowcode", "raw"], default="auto",
                    help="H2D format of the e2e leg: row-delta coded (host encode inside the "
                         "timed region), the raw int64 KJT, or auto = row-coded with the largest "
                         "keys copied raw while the host encodes the rest (share balanced "
                         "between the PCIe link and the rank's host cores)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=0,
                    help="rows in the CPU sample (0 = calibrated to --cpu-seconds)")
    ap.add_argument("--cpu-seconds", type=float, default=8.0,
                    help="target CPU work of the bounded baseline sample")
    ap.add_argument("--cpu-port", action="store_true",
                    help="CPU legs: time the oracle/ port even if baseline/_ref exists")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e/cpu)")
    args = ap.parse_args(argv)
    c = CONFIGS[args.config]
    args.batch = args.batch or c["batch"]
    args.keys = args.keys or len(c["lens"])
    args.rows = args.rows or c["rows"]
    args.dim = args.dim or c["dim"]
    args.lens = [c["lens"][i % len(c["lens"])] for i in range(args.keys)]
    args.shared_table = c["shared_table"]
    return args


# ----------------------------------------------------------------- inputs
def make_batch(args, rank, world):
    from tools.datagen import FeatureSpec, SampleCountDist, SessionConfig, generate_clustered_batch
    specs = [FeatureSpec(f"k{i}", "user_sequence", float(args.lens[i]), args.rows,
                         args.change_prob) for i in range(args.keys)]
    nsess = CONFIGS[args.config]["sessions"]
    if nsess is None or world > 1:
        nsess = int(math.ceil(args.batch * world / args.samples_per_session * 1.3)) + 64
    cfg = SessionConfig(nsess, SampleCountDist(args.dist, args.samples_per_session), 0)
    return generate_clustered_batch(cfg, specs, args.batch, row_start=rank * args.batch)


def algorithmic_bytes(B, K, D, N_kjt, N_u, U_tot, N_ids):
    """A = 8(N_kjt + BK) + 8(N_u + U_tot + BK) + 4D N_u
    + 4D BK (expanded output) + 4D BK (grad_out read) + 2*4D N_ids (SGD RMW)."""
    return (8 * (N_kjt + B * K) + 8 * (N_u + U_tot + B * K) + 4 * D * N_u + 8 * D * B * K
            + 8 * D * N_ids)


def config_dict(args):
    """Identical for both arms (the driver compares them)."""
    c = CONFIGS[args.config]
    return {"workload": c["workload"], "global_batch": args.batch * args.gpus,
            "batch_per_gpu": args.batch, "keys": args.keys, "max_len": max(args.lens),
            "tables": 1 if args.shared_table else args.keys,
            "table": f"{args.rows}x{args.dim} fp32", "samples_per_session": args.samples_per_session,
            "session_dist": args.dist, "change_prob": args.change_prob, "mode": args.mode,
            "parallelism": (f"dp{args.gpus} + row-sharded tables" if args.gpus > 1 else "single"),
            "l2": c["l2"]}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {"hbm_gbs": 6650.0, "note": "fallback (B200_PROFILING.md)"}


def load_traffic():
    """DRAM bytes per launch of the top kernels from the latest committed
    `ncu --set full` capture (profiles/traffic.json, written by
    tools/ncu_traffic.py from the .ncu-rep of the same commit)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


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
# The reference's CPU path over a bounded sample of the workload's rows.  The
# sample's records, the table and grad_out are built once in the parent; the
# pool forks after that, so workers share them read-only (the SGD'd rows go to
# a private buffer -- no copy-on-write of the shared table inside the timer).
_CPU: dict = {}


def _reference_modules():
    """The unmodified reference (`sessiondedup`) from baseline/_ref, or None."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "sessiondedup")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    from sessiondedup import tensors, trainer_sim
    return tensors, trainer_sim


def _cpu_chunk(ab):
    """Rows [a, b) of the sample, every key: the reference forward --
    build_ikjt (tensors.py:269-308), embedding_lookup + pool
    (trainer_sim.py:308-344), pooled[inverse_lookup] (558-561) -- then the
    backward restatement (oracle/embedding.py: grad_u segment-sum, ID-sorted
    reduce) and the SGD'd rows W[ids] - lr*g into a private buffer."""
    import oracle
    a, b = ab
    S = _CPU
    W = S["weights"]
    t0 = time.perf_counter()
    chk = 0.0
    for k in S["keys"]:
        if S["kind"] == "reference":
            T, TS = S["ref"]
            ik = T.build_ikjt(S["records"][a:b], [k])
            jt = ik.per_feature[k]
            acts = TS.embedding_lookup(jt, S["table"], k)
            pooled = TS.pool(acts, jt.offsets, "sum")
            out = pooled[ik.inverse_lookup]
            inv, uv, uo = ik.inverse_lookup, jt.values, jt.offsets
        else:
            v, o = S["values"][k], S["offsets"][k]
            lo = int(o[a])
            hi = int(o[b]) if b < o.size else v.size
            inv, [(uv, uo)] = oracle.build_ikjt_arrays([(v[lo:hi], o[a:b] - lo)])
            out = oracle.expand(oracle.pooled_lookup(uv, uo, W, "sum"), inv)
        gu = oracle.pool_backward(S["grad"][a:b], inv, uo.size)
        ids, gw = oracle.sparse_table_grad(gu, uv, uo, "sum")
        upd = W[ids] - (np.float32(S["lr"]) * gw).astype(np.float32)
        chk += float(out[0, 0]) + (float(upd[0, 0]) if ids.size else 0.0)
    return time.perf_counter() - t0, chk


def _pin_one_core():
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except (AttributeError, OSError):
        pass


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class CpuReference:
    """The CPU arm: a persistent fork pool over all host cores (chunks =
    split_batch of the sample, trainer_sim.py:416-446) and a one-process pool
    pinned to one core."""

    def __init__(self, args, batch, force_port=False):
        import multiprocessing as mp
        ref = None if force_port else _reference_modules()
        self.kind = "reference" if ref is not None else "port"
        self.procs = host_cores()
        self.B = batch.batch_size
        keys = list(batch.keys)
        D, rows = args.dim, args.rows
        rng = np.random.default_rng(0)
        # one table of the config's shape, shared by all keys (a 10M x 128 table
        # is 5.1 GB; the 26 tables of cfg2 would not fit the host), drawn in chunks
        w = np.empty((rows, D), np.float32)
        for r0 in range(0, rows, 1 << 20):
            r1 = min(rows, r0 + (1 << 20))
            w[r0:r1] = rng.random((r1 - r0, D), dtype=np.float32) * np.float32(0.2) - np.float32(0.1)
        _CPU.clear()
        _CPU.update(keys=keys, lr=args.lr, kind=self.kind, weights=w,
                    grad=rng.standard_normal((self.B, D), dtype=np.float32),
                    values=batch.values, offsets=batch.offsets)
        if ref is not None:
            T, TS = ref
            _CPU["ref"] = ref
            _CPU["table"] = TS.EmbeddingTable(key="shared", rows=rows, dim=D, weights=w)
            _CPU["weights"] = _CPU["table"].weights
            _CPU["records"] = self._records(batch, keys)
        ctx = mp.get_context("fork")
        self.pool = ctx.Pool(self.procs)
        self.pool1 = ctx.Pool(1, initializer=_pin_one_core)

    @staticmethod
    def _records(batch, keys):
        """The reference's input: one record (Mapping of key -> ID list) per row."""
        recs = []
        vals = {k: batch.values[k] for k in keys}
        offs = {k: np.append(batch.offsets[k], batch.values[k].size) for k in keys}
        for i in range(batch.batch_size):
            recs.append({k: vals[k][offs[k][i]:offs[k][i + 1]] for k in keys})
        return recs

    def close(self):
        self.pool.close()
        self.pool1.close()
        self.pool.join()
        self.pool1.join()

    def step(self, rows):
        """Wall seconds of one sample of `rows` rows on all cores."""
        n = max(1, min(self.procs, rows))
        q, r = divmod(rows, n)   # split_batch: the first r chunks get one more row
        bounds, a = [], 0
        for i in range(n):
            b = a + q + (1 if i < r else 0)
            bounds.append((a, b))
            a = b
        t0 = time.perf_counter()
        self.pool.map(_cpu_chunk, bounds, chunksize=1)
        return time.perf_counter() - t0

    def one_core(self, rows):
        """Seconds for `rows` rows in one process pinned to one core (after a
        warm-up call: imports, first touch of the shared table)."""
        self.pool1.apply(_cpu_chunk, ((0, min(rows, 64)),))
        return self.pool1.apply(_cpu_chunk, ((0, rows),))[0]

    def calibrate(self, target_s):
        """Rows whose all-core step takes about target_s (probe on 1,024 rows)."""
        probe = min(self.B, 1024)
        self.step(probe)
        t = self.step(probe)
        return int(max(probe, min(self.B, probe * target_s / max(t, 1e-3))))

    def describe(self, rows, procs, what):
        src = ("reference sessiondedup (baseline/_ref): build_ikjt + embedding_lookup + pool + "
               "b[inv]" if self.kind == "reference" else
               "oracle/ port of build_ikjt + lookup/pool/expand")
        return (f"first {rows} of {self.B} rows x {len(_CPU['keys'])} keys per step, {src}, then "
                f"the oracle/ backward restatement + SGD'd rows (no reference backward exists); "
                f"one shared {_CPU['weights'].shape[0]}x{_CPU['weights'].shape[1]} fp32 table; "
                f"{what}")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    batch = make_batch(args, 0, 1)
    cpu = CpuReference(args, batch, force_port=args.cpu_port)
    try:
        # each step a bounded sample, capped so the whole run fits ~3 minutes
        per_step = min(args.cpu_seconds, 150.0 / (max(1, args.steps) + 1))
        rows = args.cpu_rows or cpu.calibrate(per_step)
        for _ in range(max(0, min(args.warmup, 1))):
            cpu.step(min(rows, 1024))
        times = [cpu.step(rows) for _ in range(max(1, args.steps))]
        rows1 = max(64, min(rows, int(rows / cpu.procs)))
        t1 = cpu.one_core(rows1)
    finally:
        cpu.close()
    t = float(np.mean(times))
    value = rows / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (ids int64)", "data": "synthetic (restated reference session generator)",
        "config": config_dict(args),
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cpu.procs, "kind": cpu.kind,
                         "sample": cpu.describe(rows, cpu.procs,
                                                f"{cpu.procs} processes (persistent fork pool, "
                                                f"split_batch row chunks)"),
                         "one_core": {"value": rows1 / t1, "unit": "samples/s", "cores": 1,
                                      "sample": f"first {rows1} rows, 1 process pinned to 1 core"}},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- launcher
def spawn_ranks(args):
    """`--gpus N` without a launcher: run this script under
    torch.distributed.run with N ranks (standalone rendezvous on 127.0.0.1,
    free port chosen by the launcher) and pass its exit code through; rank
    0's stdout is the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--local-addr",
           "127.0.0.1", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "4"))
    return subprocess.call(cmd, env=env)


# ------------------------------------------------------------------- main
def main():
    args = parse()
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is not None and int(world_env) != args.gpus:
        print(json.dumps({"error": f"WORLD_SIZE={world_env} but --gpus {args.gpus}"}), flush=True)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and world_env is None:
        return spawn_ranks(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        return run_sharded(args, world, rank, local, dev)
    return run_single(args, dev)


def _unique_ids_per_table(step, keys, tables, counts, mode):
    """Distinct IDs per table among the step's unique values (the SGD RMW term)."""
    import torch
    by_table: dict = {}
    for f, k in enumerate(keys):
        n = counts.N_u[f]
        src = step.uvalues[f] if mode == "dedup" else step.in_values[f]
        by_table.setdefault(id(tables[k]), []).append(src[:n])
    return sum(int(torch.unique(torch.cat(v)).numel()) for v in by_table.values())


def run_single(args, dev):
    import torch

    import paper_2211_05239_b200 as R
    from paper_2211_05239_b200.step import TrainStep

    t_setup = time.perf_counter()
    batch = make_batch(args, 0, 1)
    keys = list(batch.keys)
    if args.shared_table:
        t = R.EmbeddingTable.create_on_device("shared", args.rows, args.dim, seed=0, device=dev)
        tables = {k: t for k in keys}
    else:
        tables = {k: R.EmbeddingTable.create_on_device(k, args.rows, args.dim, seed=i, device=dev)
                  for i, k in enumerate(keys)}
    caps = {k: batch.values[k].size for k in keys}
    pipe = args.pipeline and not (args.no_graph or args.profile)
    step = TrainStep([[k] for k in keys], args.batch, caps, tables, "sum", args.lr, args.mode, dev,
                     overlap=not args.no_overlap, slots=1 if (args.no_e2e or args.profile) else 2,
                     pipeline=pipe)
    for s_ in range(step.nslots):
        step.load_batch(batch.values, batch.offsets, slot=s_)
    step.fill_grad_out(1)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup

    # one eager step to read the step's statistics
    step.run()
    torch.cuda.synchronize()
    step.check()
    counts = step.host_counts()
    stream = torch.cuda.current_stream(dev)
    B, K, D = args.batch, len(keys), args.dim
    N_kjt = int(sum(caps.values()))
    N_u = int(sum(counts.N_u))
    U_tot = int(sum(counts.U))
    N_ids = _unique_ids_per_table(step, keys, tables, counts, args.mode)

    for _ in range(args.warmup):
        step.run()
    if not args.no_graph:
        step.capture()
    if pipe:
        step.prime(0)      # batch 0's IKJT + backward prepare; every replay then
    for i in range(max(1, args.warmup)):   # trains batch i and prepares batch i + 1
        step.replay(i % 2 if pipe else None)
    torch.cuda.synchronize()

    # ------------------------------------------------------ timed region
    sampler = ClockSampler(dev.index) if not args.profile else None
    i0 = max(1, args.warmup)
    torch.cuda.synchronize()
    launches0 = R.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        step.replay((i0 + i) % 2 if pipe else None)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    clocks = sampler.stop() if sampler else None
    step.check()
    launches_per_step = R.launch_count() - launches0
    if not args.no_graph:
        # graph replays do not pass through the host counter: count one eager step
        l0 = R.launch_count()
        if pipe:
            step.run_pipelined(0)
        else:
            step.run()
        launches_per_step = R.launch_count() - l0
        torch.cuda.synchronize()
        if pipe:
            step.use_slot(0, 0)
    value = B / (ms / 1e3)

    # --------------------------------------- per-phase timing (roofline)
    # serial, one stream (the step overlaps the occurrence sort with the lookup)
    L = R._lib
    if args.mode == "dedup" and step.fused_expand:
        calls = {"dedup": step.dedup,
                 "bwd_inverse": lambda s_: step.backward_stages(L.BWD_INVERSE, s_),
                 "pool_expand": step.forward_expand,
                 "bwd_occurrences": lambda s_: step.backward_stages(L.BWD_OCCURRENCES, s_),
                 "bwd_grad": lambda s_: step.backward_stages(L.BWD_GRAD, s_),
                 "bwd_scatter": lambda s_: step.backward_stages(L.BWD_SCATTER, s_)}
    else:
        calls = {"dedup": step.dedup, "pool": step.forward, "expand": step.expand,
                 "bwd": step.backward}
    phases = {k: [] for k in calls}
    s = stream.cuda_stream
    for _ in range(max(3, min(args.steps, 20))):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(calls) + 1)]
        ev[0].record(stream)
        for i, fn in enumerate(calls.values()):
            fn(s)
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
        for i, name in enumerate(phases):
            phases[name].append(ev[i].elapsed_time(ev[i + 1]))
    ph = {k: float(np.mean(v)) for k, v in phases.items()}
    peaks = load_peaks()
    peak = peaks.get("hbm_gbs")

    lib = R.load_library()
    nk = max(3, min(args.steps, 10))
    kernels = {}
    # compulsory HBM bytes per launch (distinct table rows once; SURVEY §8(d)
    # counts every gathered row: "requested")
    kb = {"k_pool_fwd": (8 * N_u + 8 * U_tot + 4 * D * N_ids + 4 * D * U_tot,
                         8 * N_u + 8 * U_tot + 4 * D * N_u + 4 * D * U_tot),
          "k_scatter": (8 * N_u + 4 * D * U_tot + 8 * D * N_ids,
                        8 * N_u + 4 * D * N_u + 8 * D * N_ids)}
    if args.mode == "dedup" and step.fused_expand:
        # the lookup stores every batch row itself (recd_pool_fwd_csr): out
        # rows instead of pooled rows, plus the CSR (int32 starts + rows)
        kb["k_pool_fwd"] = (8 * N_u + 8 * U_tot + 4 * D * N_ids + 4 * D * B * K + 8 * B * K,
                            8 * N_u + 8 * U_tot + 4 * D * N_u + 4 * D * B * K + 8 * B * K)
    if args.mode == "kjt":
        kb = {"k_pool_fwd": (8 * N_kjt + 4 * D * N_ids + 4 * D * B * K,
                             8 * N_kjt + 4 * D * N_kjt + 4 * D * B * K),
              "k_scatter": (8 * N_kjt + 4 * D * B * K + 8 * D * N_ids,
                            8 * N_kjt + 4 * D * N_kjt + 8 * D * N_ids)}
    for name, (comp, req) in kb.items():
        t = kernel_ms(lib, stream, name, step.run, nk)
        kernels[name] = {"ms": t, "compulsory_bytes": comp, "requested_bytes": req,
                         "achieved_gbs": comp / (t / 1e3) / 1e9,
                         "achieved_requested_gbs": req / (t / 1e3) / 1e9}
    dom = max(kernels, key=lambda k: kernels[k]["ms"])
    A = algorithmic_bytes(B, K, D, N_kjt, N_u, U_tot, N_ids)
    if args.mode == "kjt":
        A = algorithmic_bytes(B, K, D, N_kjt, N_kjt, B * K, N_ids) - 8 * (N_kjt + 2 * B * K)
    step_gbs = A / (ms / 1e3) / 1e9

    # ----------------------------------------------------------- e2e
    e2e = None
    if not args.no_e2e and not args.profile:
        if pipe:
            rc, th, sh = e2e_wire(args, 1)
            e2e = e2e_step_pipeline(step, batch, keys, dev, max(4, min(args.steps, 20)), rc, th, sh)
        else:
            rc, th, sh = e2e_wire(args, 1)
            e2e = e2e_pipelined(step, batch, keys, step.replay, dev, max(4, min(args.steps, 20)), 1,
                                rowcode=rc, threads=th, raw_share=sh)
            e2e["how"] = ("public TrainStep API: pinned-host KJT -> "
                          + ("host row-delta encode (librecd_host) -> " if rc else "") +
                          "H2D on a copy stream straight "
                          "into the step's other input slot (overlaps the previous step; one CUDA "
                          "graph per slot, value counts read on the device, no device-to-device "
                          "copy) -> graph replay -> D2H of the step's dedup counts read by the host")

    # ------------------------------------------------------ CPU baseline
    cpu = None
    if not args.no_cpu and not args.profile:
        ref = CpuReference(args, batch, force_port=args.cpu_port)
        try:
            rows = args.cpu_rows or ref.calibrate(args.cpu_seconds)
            t = ref.step(rows)
            rows1 = max(64, min(rows, int(rows / ref.procs)))
            t1 = ref.one_core(rows1)
        finally:
            ref.close()
        cpu = {"value": rows / t, "unit": "samples/s", "cores": ref.procs, "kind": ref.kind,
               "sample": ref.describe(rows, ref.procs, f"{ref.procs} processes, {t:.1f} s"),
               "one_core": {"value": rows1 / t1, "unit": "samples/s", "cores": 1,
                            "sample": f"first {rows1} rows, 1 process pinned to 1 core"}}

    traffic = load_traffic()
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (ids int64)", "data": "synthetic (restated reference session generator)",
        "config": config_dict(args),
        "roofline": roofline_entry(dom, kernels[dom], peak, peaks, traffic, args.config),
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
    return 0


def kernel_ms(lib, stream, name, run, n):
    """Average duration of one named librecd kernel, timed live with CUDA
    events that librecd records on the kernel's own stream right before /
    after its launch (recd_debug_kernel_events), over n eager steps."""
    import torch
    ts = []
    for _ in range(n):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        b.record(stream)
        lib.recd_debug_kernel_events(name.encode(), a.cuda_event, b.cuda_event)
        run()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    lib.recd_debug_kernel_events(None, None, None)
    return float(np.mean(ts))


def roofline_entry(dom, k, peak, peaks, traffic, config):
    tr = traffic.get(config, {}).get(dom) if isinstance(traffic.get(config), dict) else None
    return {"bound": "hbm", "kernel": dom, "achieved": k["achieved_gbs"], "peak": peak,
            "unit": "GB/s", "frac": k["achieved_gbs"] / peak if peak else None,
            "peak_source": ("MEASURED_PEAKS.json hbm_gbs (measured)" if "note" not in peaks
                            else peaks["note"]),
            "traffic": tr.get("dram_bytes") if tr else None,
            "traffic_source": tr.get("source") if tr else None,
            "algorithmic_bytes_per_launch": k["compulsory_bytes"],
            "bytes_definition": "compulsory: each distinct table row once (DESIGN.md §4)",
            "avg_launch_ms": k["ms"], "achieved_requested": k["achieved_requested_gbs"]}


def e2e_wire(args, world):
    """(row-coded?, encoder threads per rank, raw share) for the e2e leg.  The
    share x of the IDs that goes over PCIe raw balances the copy engine
    against the rank's encoder cores.  The copy engine carries the raw IDs and
    the coded rest (rho ~ 0.09 of its raw size: literals, codes, offsets) at
    ~47 GB/s per GPU while the host encodes; the encoder reads ~6.25 GB/s of
    KJT per core (both measured on the B200 hosts, cfg2):
    (x + rho (1 - x)) / 47 = (1 - x) / (6.25 cores)."""
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    per_rank = max(1, (cores or 1) // max(world, 1))
    if args.e2e_wire == "raw" or (args.e2e_wire == "auto" and per_rank < 8):
        # < 8 cores per rank: N = 4 on the 16-core hosts here was 9.7 M samples/s
        # row-coded vs 12.7 M raw (the ranks' copies and encoders share the host)
        return False, per_rank, 1.0
    c, e, rho = 47.0, 6.25 * per_rank, 0.09
    share = (1.0 / e - rho / c) / ((1.0 - rho) / c + 1.0 / e)
    if args.e2e_raw_share is not None:
        share = args.e2e_raw_share
    return True, per_rank, (share if args.e2e_wire == "auto" else 0.0)


def e2e_pipelined(step, batch, keys, replay, dev, n_steps, world, dist=None, rowcode=True,
                  threads=0, raw_share=0.0):
    """End-to-end samples/s through the public step API from pinned host
    buffers: every step's KJT goes H2D (copy stream, double-buffered, so the
    copy of batch i+1 overlaps step i), the step runs, and its dedup counts
    come back D2H and are read by the host (one step of lag)."""
    import torch

    from paper_2211_05239_b200.staging import H2DPipeline

    pin_v = {k: torch.from_numpy(batch.values[k]).pin_memory() for k in keys}
    pin_o = {k: torch.from_numpy(batch.offsets[k]).pin_memory() for k in keys}
    pipe = H2DPipeline(step, dev, rowcode=rowcode, threads=threads, raw_share=raw_share)
    res = [torch.empty(step.counts.numel(), dtype=torch.int64).pin_memory() for _ in range(2)]
    direct = pipe.direct
    done = [torch.cuda.Event(), torch.cuda.Event()]

    def loop(n):
        pipe.prefetch(0, pin_v, pin_o)
        for i in range(n):
            if i + 1 < n:
                pipe.prefetch((i + 1) % 2, pin_v, pin_o)
            if direct:   # the step reads the staged slot itself (one graph per slot)
                pipe.run(i % 2, replay)
            else:
                pipe.install(i % 2)
                replay()
            res[i % 2].copy_(step.counts, non_blocking=True)
            done[i % 2].record()
            if i >= 1:
                done[(i - 1) % 2].synchronize()
                _ = int(res[(i - 1) % 2][0])
        torch.cuda.synchronize()
        _ = int(res[(n - 1) % 2][0])

    loop(3)   # untimed warm-up: first touch of the staging buffers, encoder threads
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    loop(n_steps)
    e2e_s = (time.perf_counter() - t0) / n_steps
    h2d = max(pipe.h2d_bytes)
    if dist is not None:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    B = step.B
    raw = sum(pin_v[k].numel() * 8 + pin_o[k].numel() * 8 for k in keys)
    return {"value": world * B / e2e_s, "unit": "samples/s", "h2d_bytes_per_step": h2d * world,
            "d2h_bytes_per_step": res[0].numel() * 8 * world, "ms_per_step": e2e_s * 1e3,
            "h2d_gbs_per_gpu": h2d / e2e_s / 1e9,
            "wire": (f"row-delta coded: host encode ({threads or 'all'} C++ threads per rank) of "
                     f"the KJT inside the timed region, the largest keys (>= {raw_share:.2f} of the "
                     "IDs) copied raw meanwhile; "
                     f"{raw / max(h2d, 1):.1f}x fewer H2D bytes than the raw "
                     "int64 KJT, device decode on the copy stream") if rowcode else "raw int64 KJT"}


def e2e_step_pipeline(step, batch, keys, dev, n_steps, rowcode=True, threads=0, raw_share=0.0):
    """End to end through the pipelined TrainStep: batch i+2 goes H2D (copy
    stream, pinned host) into the slot batch i came in while graph i trains
    batch i and deduplicates batch i+1 on its side stream; each step's dedup
    counts come back D2H and are read by the host (one step of lag).  Every
    batch is copied, deduplicated and trained inside the timed region."""
    import torch

    from paper_2211_05239_b200.staging import H2DPipeline

    pin_v = {k: torch.from_numpy(batch.values[k]).pin_memory() for k in keys}
    pin_o = {k: torch.from_numpy(batch.offsets[k]).pin_memory() for k in keys}
    pipe = H2DPipeline(step, dev, rowcode=rowcode, threads=threads, raw_share=raw_share)
    res = [torch.empty(step.counts.numel(), dtype=torch.int64).pin_memory() for _ in range(2)]
    done = [torch.cuda.Event(), torch.cuda.Event()]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pipe.prefetch(0, pin_v, pin_o)
    pipe.prefetch(1, pin_v, pin_o)
    pipe.wait_ready(0)
    step.prime(0)
    for i in range(n_steps):
        p = i % 2
        pipe.wait_ready(1 - p)      # batch i+1: deduplicated by this graph's side stream
        pipe.release(p)             # batch i's slot was consumed by the previous graph
        step.replay(p)
        if i + 2 <= n_steps:        # batch i+2 into the freed slot, overlapping this graph
            pipe.prefetch(p, pin_v, pin_o)
        res[p].copy_(step.counts, non_blocking=True)
        done[p].record()
        if i >= 1:
            done[1 - p].synchronize()
            _ = int(res[1 - p][0])
    torch.cuda.synchronize()
    _ = int(res[(n_steps - 1) % 2][0])
    e2e_s = (time.perf_counter() - t0) / n_steps
    h2d = max(pipe.h2d_bytes)
    return {"value": step.B / e2e_s, "unit": "samples/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": res[0].numel() * 8, "ms_per_step": e2e_s * 1e3,
            "h2d_gbs_per_gpu": h2d / e2e_s / 1e9,
            "how": "public TrainStep(pipeline=True) API: pinned-host KJT -> H2D on a copy stream "
                   "into the slot the batch two steps back came in (overlaps the step) -> one graph "
                   "per step parity (batch i's lookup/expand/backward + SGD, batch i+1's dedup + "
                   "backward prepare on a side stream) -> D2H of the step's dedup counts"}


def run_sharded(args, world, rank, local, dev):
    """N > 1: every table row-sharded into S shards (id mod S), the
    (table, shard) pairs placed on ranks LPT-first, + data-parallel batch;
    each rank deduplicates its own 65,536-row chunk of the global batch and
    the exchange carries only deduplicated IDs, partially pooled rows and
    unique-row gradients (peer.py over NVLink peer memory, or sharded.py over
    NCCL)."""
    import torch
    import torch.distributed as dist

    import paper_2211_05239_b200 as R
    from paper_2211_05239_b200.peer import PeerShardedStep, _DevArray
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
    ms_rank = e0.elapsed_time(e1) / args.steps
    clocks = sampler.stop() if sampler else None
    launches_per_step = (R.launch_count() - launches0) // max(args.steps, 1)
    t = torch.tensor([ms_rank], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = world * B / (ms / 1e3)

    # sub-phase breakdown (one traced step per rank; max over ranks + per rank)
    step.trace = True
    l0 = R.launch_count()
    step.run()
    if peer:   # graph replays do not pass through the host counter: count this eager step
        launches_per_step = R.launch_count() - l0
    ph = step.phase_ms()
    step.trace = False
    names = list(ph)
    tph = torch.tensor([ph[n] for n in names], device=dev)
    allph = [torch.empty_like(tph) for _ in range(world)]
    dist.all_gather(allph, tph)
    ph_max = dict(zip(names, torch.stack(allph).max(0).values.tolist()))
    ph_rank = [dict(zip(names, x.tolist())) for x in allph]

    # ------------------------------------------------ roofline (per rank)
    # The SURVEY §8(d) step bytes of this rank's local batch (dedup, gather,
    # expand, grad read) + the SGD RMW of the distinct rows this rank OWNS
    # (the rows it received from every source); the dominant kernel is the
    # owner's sorted scatter + SGD (k_scatter), timed live like at N = 1.
    N_kjt = int(sum(caps.values()))
    Nu_r, U_r = int(sum(N_u)), int(sum(U))
    own_rows = own_ids = own_distinct = 0
    if peer and step.Q:
        oc = step.ctl[step.i_own_counts:step.i_own_counts + 2 * step.Q].cpu().tolist()
        own_rows, own_ids = sum(oc[:step.Q]), sum(oc[step.Q:])
        for q in range(step.Q):
            n = int(oc[step.Q + q])
            if n:
                ids = torch.as_tensor(_DevArray(step._peer(rank, "ids", q), n, "<i8"), device=dev)
                own_distinct += int(torch.unique(ids).numel())
    A_r = (8 * (N_kjt + B * K) + 8 * (Nu_r + U_r + B * K) + 4 * D * Nu_r + 8 * D * B * K
           + 8 * D * own_distinct)
    sc_bytes = 8 * own_ids + 4 * D * own_rows + 8 * D * own_distinct
    lib = R.load_library()
    sc_ms = kernel_ms(lib, stream, "k_scatter", step.run, 3) if (peer and step.Q) else 0.0
    vec = torch.tensor([A_r, ms_rank, sc_bytes, sc_ms, own_distinct, Nu_r, U_r], dtype=torch.float64,
                       device=dev)
    allv = [torch.empty_like(vec) for _ in range(world)]
    dist.all_gather(allv, vec)
    per = torch.stack(allv).cpu().numpy()
    peaks = load_peaks()
    peak = peaks.get("hbm_gbs")

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

    e2e = None
    if not args.no_e2e and not args.profile:
        rc, th, sh = e2e_wire(args, world)
        e2e = e2e_pipelined(step, batch, keys, step.replay if peer else step.run, dev,
                            max(4, min(args.steps, 10)), world, dist, rowcode=rc, threads=th,
                            raw_share=sh)
        e2e["how"] = (f"{cls.__name__} on every rank: pinned-host KJT -> H2D on a copy stream "
                      "(double-buffered) -> step -> D2H of the dedup counts; max over ranks")
    if rank == 0:
        A_job = float(per[:, 0].sum())
        job_gbs = A_job / (ms / 1e3) / 1e9 / world     # per-GPU average
        ach = [b / (m / 1e3) / 1e9 if m > 0 else 0.0 for b, m in zip(per[:, 2], per[:, 3])]
        r0 = int(np.argmax(per[:, 3]))                 # slowest owner scatter
        roof = {"bound": "hbm", "kernel": "k_scatter (owner sorted scatter-add + SGD)",
                "achieved": ach[r0], "peak": peak, "unit": "GB/s",
                "frac": ach[r0] / peak if peak else None,
                "peak_source": ("MEASURED_PEAKS.json hbm_gbs (measured)" if "note" not in peaks
                                else peaks["note"]),
                "traffic": None, "algorithmic_bytes_per_launch": float(per[r0, 2]),
                "avg_launch_ms": float(per[r0, 3]), "rank": r0,
                "bytes_definition": "8 n_ids_received + 4D rows_received + 2*4D distinct owned "
                                    "rows (compulsory)",
                "per_rank_frac": [a / peak for a in ach] if peak else None}
        step_roof = {"algorithmic_bytes_job": A_job,
                     "achieved_gbs_per_gpu": job_gbs, "frac": job_gbs / peak if peak else None,
                     "per_rank_frac": [float(a / (m / 1e3) / 1e9 / peak) for a, m in
                                       zip(per[:, 0], per[:, 1])] if peak else None,
                     "definition": "sum over ranks of SURVEY §8(d) A on the rank's local batch, "
                                   "with N_ids = distinct rows each owner updates; / (N x max-rank "
                                   "step time)"}
        a2a_fwd_dedup = sum(16 + 8 * (U[f] + N_u[f]) for f in range(len(keys)))
        a2a_fwd_kjt = sum(16 + 8 * (args.batch + int(caps[k])) for k in keys)
        a2a = {"fwd_bytes_dedup": a2a_fwd_dedup, "fwd_bytes_kjt": a2a_fwd_kjt,
               "fwd_reduction": a2a_fwd_kjt / max(a2a_fwd_dedup, 1),
               "back_bytes_dedup": 4 * D * int(sum(U)), "back_bytes_kjt": 4 * D * args.batch * len(keys),
               "definition": "trainer_sim.sdd / a2a_bytes_back (trainer_sim.py:281-305, 557, 573) on "
                             "rank 0's batch; the inverse never travels"}
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 (ids int64)", "data": "synthetic (restated reference session generator)",
            "config": config_dict(args),
            "sharding": {"shards_per_table": S, "shard_of_id": f"id mod {S}",
                         "placement": "(table, shard) pairs LPT over ranks",
                         "transport": ("NVLink peer memory (CUDA IPC), whole step one CUDA graph"
                                       if peer else "NCCL all-to-all, host-planned split sizes"),
                         "table_rows_rank0": lrows, "pairs_rank0": len(step.mine)},
            "roofline": roof, "step_roofline": step_roof,
            "phases_ms": ph_max, "phases_ms_per_rank": ph_rank,
            "ms_per_step_per_rank": [float(x) for x in per[:, 1]],
            "comm_bytes_sent_rank0": sent, "a2a_accounting_rank0": a2a,
            "stats_rank0": {"N_kjt": N_kjt, "N_u": Nu_r, "U_tot": U_r},
            "cpu_baseline": None, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps * world,
            "gpu_launches_per_step_per_rank": launches_per_step, "clocks": clocks,
            "setup_s": setup_s,
        }
        print(json.dumps(line), flush=True)
    if peer:
        step.close()
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
