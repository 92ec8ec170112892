#!/usr/bin/env python3
"""GN engine benchmark: GN edge-updates/s (undirected edges x iterations / s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step is one run_wrgn over one instance: the reference's default pursuit
schedule (linear gamma 0.9 -> 1.5, 1000 iterations, dynamics.py:58-63) on the
workload BASELINE.json's metric is quoted on at one GPU -- configs[1], the
256x256 assignment conflict graph (C2), fp32 gathered values.  N > 1: one
process per GPU (torchrun), each rank runs its own replica (C2 does not
shard: "replicas only"), `value` counts all ranks' edge updates
over the max-over-ranks device time.  --config C4 shards the C4 batch instead
(1024 graphs per rank, no collectives).

Printed JSON keys follow the driver contract; see DESIGN.md "Measurement".
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402

METRIC = "GN edge-updates/sec (edges x iters / s)"
UNIT = "edge-updates/s"

CONFIG_TEXT = {
    "C1": "Erdos-Renyi G(n=1000, avg degree 10), w ~ U(0,1], fp64, init_random x0, pursuit 0.9->1.5 x1000",
    "C2": "assignment-as-MWIS: conflict graph of a 256x256 assignment (65,536 vertices, 16,711,680 edges), "
          "w ~ U(0,1] fp32, pursuit 0.9->1.5 x1000",
    "C3": "Barabasi-Albert n=200,000 m=5 (999,975 edges), integer weights U{1..200} fp64, pursuit x1000",
    "C4": "1024 independent ER graphs n=2000 avg degree 16 per GPU, packed block-diagonal, fp32, pursuit x1000",
    "C5": "R-MAT edge factor 16 (a=.57,b=c=.19), symmetrised, dedup, fp32, pursuit x1000 (scale in config.scale)",
}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_instance(config: str, rank: int, scale: int):
    from paper_2605_05330_b200 import generators as G

    if config == "C1":
        return G.c1_er()
    if config == "C2":
        return G.c2_assignment()
    if config == "C3":
        return G.c3_ba()
    if config == "C4":
        return G.c4_batch(graphs=1024, first=rank * 1024).instance
    if config == "C5":
        return G.c5_rmat_gpu(scale) if scale >= 18 else G.c5_rmat(scale)
    raise SystemExit(f"unknown config {config}")


def algorithmic_bytes(n: int, nnz: int, s: int) -> int:
    """B_iter = 4 nnz + P (n+1) + 3 s n (P = 4 below 2^31 entries)."""
    p = 4 if nnz < 2**31 else 8
    return 4 * nnz + p * (n + 1) + 3 * s * n


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def flush_l2(torch, dev):
    """Write a buffer larger than the 126 MB L2 between timed steps."""
    buf = getattr(flush_l2, "buf", None)
    if buf is None:
        buf = flush_l2.buf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    buf.fill_(1)


def cpu_reference(inst, seconds: float = 12.0, threads: int | None = None) -> dict:
    """The CPU path (oracle port of the reference, fp64, all host threads) on
    a bounded sample of the same workload: the first S pursuit iterations."""
    import gn_oracle as O
    from paper_2605_05330_b200 import GammaSchedule

    threads = threads or O.default_threads()
    tab = GammaSchedule.pursuit().table()
    t0 = time.perf_counter()
    O.run(inst.graph, inst.x0, tab[:2], 1.5, threads=threads)
    per = max((time.perf_counter() - t0) / 2, 1e-6)
    k = int(min(1000, max(2, seconds / per)))
    t0 = time.perf_counter()
    O.run(inst.graph, inst.x0, tab[:k], 1.5, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": inst.m * k / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"first {k} of the 1000 pursuit iterations of {inst.name} in fp64 "
                      f"(oracle/gn_oracle.c, OpenMP row-parallel, bitwise the reference), {dt:.2f} s",
            "iters": k, "seconds": dt}


def ncu_traffic(config: str, iters: int):
    """DRAM bytes (read + write) per launch of `iters` iterations, from the
    committed ncu --set full summary of the same kernel (scaled by iterations
    when the capture ran fewer, e.g. 5 iterations of C5)."""
    f = ROOT / "profiles" / "ncu_summary.json"
    if f.exists():
        try:
            d = json.loads(f.read_text()).get(config, {})
            if d.get("dram_bytes_per_launch") is None:
                return None
            return d["dram_bytes_per_launch"] / (d.get("iters_per_launch") or iters) * iters
        except Exception:
            return None
    return None


def run_reference(args, ws, rank):
    if rank != 0:
        return 0
    inst = make_instance(args.config, 0, args.scale)
    vals = []
    base = None
    for i in range(args.warmup + args.steps):
        r = cpu_reference(inst, seconds=args.ref_seconds)
        if i >= args.warmup:
            vals.append(r["value"])
            base = r
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config + ": " + CONFIG_TEXT[args.config], "n": inst.n, "m": inst.m},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": base["cores"], "kind": base["kind"],
                         "sample": base["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_partitioned(args, ws, rank, local, inst, torch, P, E) -> int:
    """C5 as BASELINE names it: the graph vertex-range partitioned over the N
    ranks (partition.py), each rank stepping its owned rows (gn_part_step) and
    exchanging boundary values with its peers every iteration: the boundary
    kernel's direct stores into the peers' ghost slots over NVLink (--halo
    peer, the default) or NCCL point-to-point through torch.distributed
    (--halo nccl).  Strong scaling: the graph is
    the same at every N.  Timed with CUDA events on the stream the engine and
    NCCL share, max over ranks."""
    from paper_2605_05330_b200.partition import (DistExchange, DistPeerExchange, EngineBackend, build_partitions,
                                                 partitioned_step)

    dtype = args.dtype or inst.dtype
    sched = P.GammaSchedule.pursuit(iterations=args.iters)
    gam = sched.table()
    iters = len(gam)
    spec = build_partitions(inst.graph, ws)[rank]
    be = EngineBackend(spec, dtype=dtype, device=local)
    # the halo: direct stores into the peers' ghost slots over NVLink (CUDA IPC
    # mappings, the default) or pack + NCCL send/recv + unpack (--halo nccl)
    ex = (DistPeerExchange(be) if args.halo == "peer" else DistExchange(be)) if ws > 1 else None
    x0l = spec.local_x0(inst.x0)
    dev = torch.device("cuda", local)

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()

    def step():
        be.begin(x0l, gam)
        if ex is not None:
            ex.setup()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(iters):
            if ex is not None:
                partitioned_step(be, ex, k)
            else:
                be.step(k)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for _ in range(args.warmup):
        flush_l2(torch, dev)
        step()
    launches0 = E.launch_count()
    times = []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush_l2(torch, dev)
            barrier()
            times.append(step())
    launches = E.launch_count() - launches0
    total_ms = float(sum(times))
    # e2e: host x0 in, the owned x out, every step (begin .. end)
    e2e = []
    for _ in range(args.steps):
        barrier()
        t0 = time.perf_counter()
        be.begin(x0l, gam)
        if ex is not None:
            ex.setup()
        for k in range(iters):
            if ex is not None:
                partitioned_step(be, ex, k)
            else:
                be.step(k)
        be.end(iters)
        barrier()
        e2e.append(time.perf_counter() - t0)
    e2e_total = sum(e2e)
    if ws > 1:
        t = torch.tensor([total_ms, e2e_total], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms, e2e_total = float(t[0].item()), float(t[1].item())
    if rank == 0:
        m, n = inst.m, inst.graph.n
        value = m * iters * args.steps / (total_ms * 1e-3)
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
        peak = float(peaks.get("hbm_gbs", 6650.0))
        s_bytes = 8 if dtype == "fp64" else 4
        b_iter = algorithmic_bytes(n, 2 * m, s_bytes)
        achieved = b_iter * iters * args.steps / (total_ms * 1e-3) / 1e9
        clk = clocks.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": {"fp64": "f64", "fp32": "f32-gather/f64-state", "fp32_pure": "f32"}[dtype],
            "data": "synthetic (seeded generators, paper_2605_05330_b200/generators.py)",
            "config": {"workload": "C5: " + CONFIG_TEXT["C5"] + f"; vertex-range partitioned over {ws} GPU(s)",
                       "n": n, "m": m, "iters": iters, "scale": args.scale, "parallelism": f"partition x{ws}",
                       "ghosts_rank0": spec.n_ghost, "owned_rank0": spec.n_own,
                       "l2": "flushed between steps (256 MB write)", "engine_dtype": dtype},
            "e2e": {"value": m * iters * args.steps / e2e_total, "unit": UNIT,
                    "h2d_bytes_per_step": 8 * (spec.n_own + spec.n_ghost) + 8 * iters,
                    "d2h_bytes_per_step": 8 * spec.n_own + 32 * iters,
                    "api": "partition.EngineBackend begin/step/halo/end (host x0 in, owned x out), rank 0 shown"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * ws, "unit": "GB/s",
                         "frac": achieved / (peak * ws), "traffic": None,
                         "kernel": "gn::k_part_step (one launch per iteration and part)" + (
                             "" if ws == 1 else (" + direct peer halo (stores into peer ghost slots, CUDA IPC)"
                                                 if args.halo == "peer" else " + NCCL halo")),
                         "b_iter": b_iter, "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs) x n_gpus"},
            "cpu_baseline": None,
            "clocks": {k: clk[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
            "gpu_launches": int(launches),
        }
        print(json.dumps(line), flush=True)
    if ex is not None and hasattr(ex, "close"):
        barrier()  # no peer still writes into our buffers
        ex.close()
    be.close()
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--scale", type=int, default=24, help="R-MAT scale for C5 (BASELINE: 24)")
    ap.add_argument("--dtype", default=None, help="engine dtype (default: fp64 for C1-C3, fp32 for C4/C5)")
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--ref-seconds", type=float, default=4.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--halo", choices=["peer", "nccl"], default="peer",
                    help="C5 under torchrun: direct stores into the peers' ghost slots (default) or NCCL send/recv")
    ap.add_argument("--partition", action="store_true",
                    help="C5: vertex-range partitioned engine (the default for C5 under torchrun, N>1)")
    ap.add_argument("--starts", type=int, default=1,
                    help="starts per instance (SURVEY 8f f1): >1 runs them together through gn_multi_run")
    args = ap.parse_args()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, ws, rank)

    import torch

    import paper_2605_05330_b200 as P
    from paper_2605_05330_b200 import _engine as E

    E.load_library()
    if E.device_count() < 1:
        raise SystemExit("bench.py needs a CUDA device (the engine has no CPU path)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    if args.config == "C4":
        from paper_2605_05330_b200 import generators as G
        from paper_2605_05330_b200.batch import GraphBatch
        from paper_2605_05330_b200.parallel import shard_range

        lo, hi = shard_range(1024 * ws, ws, rank)
        batch = G.c4_batch(graphs=hi - lo, first=lo)
        inst = batch.instance
    else:
        inst = make_instance(args.config, rank, args.scale)
        batch = None
    g = inst.graph
    if args.config == "C5" and (ws > 1 or args.partition):
        return run_partitioned(args, ws, rank, local, inst, torch, P, E)
    # C2's graph stays in L2, so binary64 gathers cost no bandwidth and avoid
    # the fp32->fp64 conversions of the mixed dtype: run it in the reference's
    # own arithmetic
    dtype = args.dtype or ("fp64" if args.config in ("C1", "C2", "C3") else inst.dtype)
    sched = P.GammaSchedule.pursuit(iterations=args.iters)
    gam = np.ascontiguousarray(sched.table())
    iters = len(gam)
    starts = max(1, args.starts) if batch is None else 1
    x0s = inst.x0[None, :] if starts == 1 else np.stack([P.init_random(g.n, [2605, b]) for b in range(starts)])
    x0_dev = torch.from_numpy(np.ascontiguousarray(x0s)).to(dev)
    x_out = torch.empty((starts, g.n), dtype=torch.float64, device=dev)
    si = np.zeros(iters)
    fb = np.zeros(iters, dtype=np.int64)
    mass = np.zeros(iters)
    ran = E.ctypes.c_int()
    fail = E.ctypes.c_int()
    flags = E.GN_DEVICE_IO
    if batch is not None:
        gb = GraphBatch(g, batch.offsets, dtype=dtype, device=local)
        kernel_name = "gn::k_gn_batch (one CTA per graph, graph resident in shared memory)"

        def device_step():
            r = gb.run(None, sched, device_x0=x0_dev.data_ptr(), device_x_out=x_out.data_ptr(), traces=False)
            st = E.RunStats()
            for f, _ in E.RunStats._fields_:
                setattr(st, f, r.stats[f])
            return st
    elif starts > 1:
        h = g.device_graph(dtype, local)
        kernel_name = "gn::k_gn_multi (persistent, all starts and iterations in 1 launch)"
        msi = np.zeros((starts, iters))
        mfb = np.zeros((starts, iters), dtype=np.int64)
        mran = np.zeros(starts, dtype=np.int32)
        mst = np.zeros(starts, dtype=np.int32)
        mfail = np.zeros(starts, dtype=np.int32)

        def device_step():
            st = E.RunStats()
            E.check(E.lib().gn_multi_run(h.handle, starts, E.ctypes.c_void_p(x0_dev.data_ptr()), E.ptr(gam), iters,
                                         1.5, flags, E.ctypes.c_void_p(x_out.data_ptr()), E.ptr(msi), E.ptr(mfb),
                                         E.ptr(mran), E.ptr(mst), E.ptr(mfail), E.ctypes.byref(st)))
            return st
    else:
        h = g.device_graph(dtype, local)
        kernel_name = "gn::k_gn_loop (persistent, 1 launch = all iterations)"

        def device_step():
            st = E.RunStats()
            E.check(E.lib().gn_run(h.handle, E.ctypes.c_void_p(x0_dev.data_ptr()), E.ptr(gam), iters, 1.5, flags,
                                   E.ctypes.c_void_p(x_out.data_ptr()), E.ptr(si), E.ptr(fb), E.ptr(mass), None, None,
                                   None, E.ctypes.byref(ran), E.ctypes.byref(fail), E.ctypes.byref(st)))
            return st

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        flush_l2(torch, dev)
        device_step()
    barrier()
    launches0 = E.launch_count()
    step_ms, loop_ms = [], []
    wall0 = time.perf_counter()
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush_l2(torch, dev)
            torch.cuda.synchronize()
            st = device_step()
            step_ms.append(st.total_ms)
            loop_ms.append(st.loop_ms)
    barrier()
    wall = time.perf_counter() - wall0
    launches = E.launch_count() - launches0
    total_ms = float(sum(step_ms))
    if ws > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    edges_all = inst.m * ws * starts
    value = edges_all * iters * args.steps / (total_ms * 1e-3)

    # ---- e2e through the public API: host x0 in, MIS out, every step.
    # The harness has torch loaded (millions of tracked objects): move them
    # out of the collector's way so a full collection cannot land in a step.
    gc.collect()
    gc.freeze()
    x0_host = torch.from_numpy(np.ascontiguousarray(inst.x0)).pin_memory().numpy()
    e2e_t, round_t = [], []
    h2d = d2h = 0
    for i in range(args.warmup + args.steps):
        barrier()
        t0 = time.perf_counter()
        if batch is not None:
            r = gb.run(x0_host, sched)
        elif starts > 1:
            r = P.run_multi(g, x0s, sched, dtype=dtype, device=local)
        else:
            r = P.run_engine(g, x0_host, sched, dtype=dtype, device=local)
        t1 = time.perf_counter()
        sol = P.round_many(g, r.x) if starts > 1 else P.round_to_mis(g, r.x)
        barrier()
        if os.environ.get("GN_BENCH_VERBOSE"):
            print(f"e2e step {i}: run {1e3 * (t1 - t0):.2f} ms, round {1e3 * (time.perf_counter() - t1):.2f} ms, "
                  f"call {r.stats['total_ms']:.2f} ms loop {r.stats['loop_ms']:.2f} ms", file=sys.stderr, flush=True)
        if i >= args.warmup:
            e2e_t.append(time.perf_counter() - t0)
            round_t.append(time.perf_counter() - t1)
            h2d = r.stats["h2d_bytes"] + 8 * g.n * starts          # + the rounding's state upload
            # + the rounding's output: member ids (round_to_mis) or membership masks (round_many), and flags
            d2h = r.stats["d2h_bytes"] + (8 * len(sol._idx) + 64 if starts == 1 else (g.n + 64) * starts)
    del sol
    e2e_total = sum(e2e_t)
    if ws > 1:
        t = torch.tensor([e2e_total], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = edges_all * iters * args.steps / e2e_total

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return 0

    peaks = {}
    pf = ROOT / "MEASURED_PEAKS.json"
    if pf.exists():
        peaks = json.loads(pf.read_text())
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    s_bytes = 8 if dtype == "fp64" else 4  # s = element size of the state vectors
    # SURVEY 8(d) per iteration; with several starts the index stream is read
    # once for all of them and the state streams once per start
    b_iter = algorithmic_bytes(g.n, 2 * inst.m, s_bytes) + 3 * s_bytes * g.n * (starts - 1)
    loop_avg = statistics.mean(loop_ms)
    achieved = b_iter * iters / (loop_avg * 1e-3) / 1e9
    traffic = ncu_traffic(args.config, iters) if starts == 1 else None
    if traffic is None:
        traffic_note = None
    elif traffic < 0.5 * b_iter * iters:
        traffic_note = (f"DRAM traffic is {traffic / (b_iter * iters):.3f}x the algorithmic bytes: the graph stays in "
                        "L2/shared memory across the iterations of a launch, so achieved/frac are the algorithmic "
                        "rate of SURVEY 8(d), not DRAM bandwidth")
    else:
        traffic_note = (f"DRAM traffic is {traffic / (b_iter * iters):.2f}x the algorithmic bytes (index stream plus "
                        "L2 misses of the gathered values)")
    info = {"n": g.n}

    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference(inst, seconds=args.ref_seconds)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}

    clk = clocks.summary()
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": {"fp64": "f64", "fp32": "f32-gather/f64-state", "fp32_pure": "f32"}[dtype],
        "data": "synthetic (seeded generators, paper_2605_05330_b200/generators.py)",
        "config": {
            "workload": args.config + ": " + CONFIG_TEXT[args.config] + (f"; {starts} starts per call" if starts > 1 else ""),
            "n": g.n, "m": inst.m, "iters": iters, "schedule": "pursuit 0.9->1.5",
            "scale": args.scale if args.config == "C5" else None,
            "parallelism": f"replicas x{ws}" if args.config != "C4" else f"batch shard x{ws} (1024 graphs/rank)",
            "l2": "flushed between steps (256 MB write); the 1000 iterations inside a step re-read the graph",
            "index_format": "uint16" if info["n"] <= 65536 else "int32",
            "inputs": "w and x0 binary32-representable (BASELINE configs[1]: fp32 weights)",
            "engine_dtype": dtype,
            "starts": starts,
        },
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "api": ("paper_2605_05330_b200.run_multi + round_many" if starts > 1 else
                        "paper_2605_05330_b200.run_engine + round_to_mis") + " (host numpy in, MIS out)",
                "round_ms_per_step": 1e3 * statistics.mean(round_t) if round_t else None},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": kernel_name,
                     "bytes_per_launch": b_iter * iters, "b_iter": b_iter, "peak_source": peak_src,
                     "loop_ms": loop_avg, "traffic_note": traffic_note},
        "cpu_baseline": cpu,
        "clocks": {k: clk[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
        "gpu_launches": int(launches),
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
