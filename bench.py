#!/usr/bin/env python3
"""GN engine benchmark: GN edge-updates/s (undirected edges x iterations / s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]

A step is one run_wrgn over one instance: the reference's default pursuit
schedule (linear gamma 0.9 -> 1.5, 1000 iterations, dynamics.py:58-63).

Default workload: BASELINE config C5 (R-MAT scale 24, 16.8 M vertices,
260 M edges, fp32 weights, fp64 arithmetic) through the vertex-range partitioned
engine: one part per GPU, every iteration from a device-side schedule (one
CUDA-graph launch per run), the halo between parts pushed over NVLink into
the peers' ghost slots (--halo peer) or exchanged by NCCL (--halo nccl).
N = 1 is one part (no halo); N > 1 is strong scaling of the same graph.
`--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one process per GPU).

Other configs: --config C2 (the 256x256 assignment conflict graph, the
persistent loop kernel; replicas at N > 1), C4 (1024 graphs per rank, batch
kernel, no collectives), C1/C3 (replicas), --config C5 --engine loop (the
single-GPU persistent loop kernel).

Printed JSON keys follow the driver contract; see DESIGN.md "Measurement".
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import socket
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
    "C5": "R-MAT scale 24 (16.8M vertices), edge factor 16 (a=.57,b=c=.19), symmetrised, dedup, w ~ U(0,1] fp32, "
          "pursuit 0.9->1.5 x1000, vertex-range partitioned over the GPUs with a per-iteration halo",
}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def spawn_ranks(n: int) -> int:
    """`--gpus N` outside torchrun: re-run this command as N ranks (one
    process per GPU) under torch.distributed.run on 127.0.0.1."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def make_instance(config: str, rank: int, ws: int, scale: int):
    from paper_2605_05330_b200 import generators as G

    if config == "C1":
        return G.c1_er(), None
    if config == "C2":
        return G.c2_assignment(), None
    if config == "C3":
        return G.c3_ba(), None
    if config == "C4":
        from paper_2605_05330_b200.parallel import shard_range

        lo, hi = shard_range(1024 * ws, ws, rank)
        batch = G.c4_batch(graphs=hi - lo, first=lo)
        return batch.instance, batch
    if config == "C5":
        return (G.c5_rmat_gpu(scale) if scale >= 18 else G.c5_rmat(scale)), None
    raise SystemExit(f"unknown config {config}")


def algorithmic_bytes(n: int, nnz: int, s: int) -> int:
    """B_iter = 4 nnz + P (n+1) + 3 s n (P = 4 below 2^31 entries)."""
    p = 4 if nnz < 2**31 else 8
    return 4 * nnz + p * (n + 1) + 3 * s * n


def engine_dtype(args, inst) -> str:
    # C1-C3 and C5 run in the reference's own arithmetic (fp64: C2's graph
    # stays in L2, so binary64 gathers cost no bandwidth; on C5 at scale 24
    # binary32 gathered values miss the per-iteration 1e-4 gate at a few
    # transition iterations -- profiles/r02_fp32_excursions -- for ~10% more
    # time, so the benched mode is fp64); C4 gathers binary32 values
    # (bitwise its same-arithmetic oracle, within the fp32 gate)
    return args.dtype or ("fp32" if args.config == "C4" else "fp64")


def config_dict(args, inst, ws: int, dtype: str, extra: dict | None = None) -> dict:
    """The workload description both arms print (same keys, same values)."""
    part = args.config == "C5" and args.engine == "part"
    d = {
        "workload": args.config + ": " + CONFIG_TEXT[args.config] + (
            f"; {args.starts} starts per call" if args.starts > 1 else ""),
        "n": int(inst.n), "m": int(inst.m), "iters": int(args.iters), "schedule": "pursuit 0.9->1.5",
        "scale": args.scale if args.config == "C5" else None,
        "parallelism": (f"partition x{ws}" if part else
                        f"batch shard x{ws} (1024 graphs/rank)" if args.config == "C4" else f"replicas x{ws}"),
        "engine": (("partitioned (gn_part_run: device-side schedule" +
                    (f", {args.halo} halo)" if ws > 1 else ", one part)")) if part else
                   "batch (gn_batch_run)" if args.config == "C4" else
                   "multi-start (gn_multi_run)" if args.starts > 1 else "loop (gn_run)"),
        "engine_dtype": dtype,
        "starts": args.starts,
        "l2": "flushed between steps (256 MB write); the iterations inside a step re-read the graph",
        "index_format": "uint16" if inst.n <= 65536 and not part else "int32",
        "inputs": "w and x0 binary32-representable (BASELINE: fp32 weights)",
    }
    if extra:
        d.update(extra)
    return d


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


# ---------------------------------------------------------------- CPU arms

_CPU_WARM: set = set()


def cpu_port(inst, seconds: float, threads: int) -> dict:
    """The oracle port (oracle/gn_oracle.c: the reference's fp64 arithmetic,
    bitwise; rows in fixed 4096-row chunks over `threads` OpenMP threads) on
    a bounded sample: the first k pursuit iterations of the same instance."""
    import gn_oracle as O
    from paper_2605_05330_b200 import GammaSchedule

    tab = GammaSchedule.pursuit().table()
    key = (id(inst), threads)
    if key not in _CPU_WARM:  # first touch of the graph's pages and the threads: not timed
        O.run(inst.graph, inst.x0, tab[:1], 1.5, threads=threads)
        _CPU_WARM.add(key)
    # the loop's own rate: T(k) - T(1) over k - 1 iterations, so the call's fixed
    # part (the x0 check's SpMV, the array hand-over) is not charged to the
    # iterations -- the GPU arm's `value` times the loop alone as well
    t0 = time.perf_counter()
    O.run(inst.graph, inst.x0, tab[:1], 1.5, threads=threads)
    t1 = time.perf_counter() - t0
    k = int(min(1000, max(3, seconds / max(t1, 1e-6))))
    t0 = time.perf_counter()
    O.run(inst.graph, inst.x0, tab[:k], 1.5, threads=threads)
    tk = time.perf_counter() - t0
    if tk - t1 < seconds / 2 and k < 1000:  # T(1) was mostly set-up: a sample of the asked length
        k = int(min(1000, max(k + 1, (k - 1) * seconds / max(tk - t1, 1e-6))))
        t0 = time.perf_counter()
        O.run(inst.graph, inst.x0, tab[:k], 1.5, threads=threads)
        tk = time.perf_counter() - t0
    dt = tk - t1
    if dt <= 0.05 * tk:  # a run too short to separate: charge everything
        dt, per_k = tk, k
    else:
        per_k = k - 1
    return {"value": inst.m * per_k / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"iterations 2..{k} of the 1000 pursuit iterations of {inst.name} in fp64 on {threads} host "
                      f"thread(s) (oracle/gn_oracle.c, OpenMP over fixed row chunks, bitwise the reference's "
                      f"arithmetic): T({k}) - T(1) = {dt:.2f} s (T(1) = {t1:.2f} s holds the x0 check and the "
                      f"call's set-up)",
            "iters": per_k, "seconds": dt}


def reference_module():
    """The unmodified reference package: baseline/_ref (installed with pip
    --target, travels to the GPU box) or, in the build container, its source
    tree.  None when neither is importable."""
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "graphnorm" / "dynamics.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            try:
                import graphnorm.dynamics as D
                import graphnorm.graph as RG

                return D, RG, str(p)
            except Exception:
                return None
    return None


def cpu_reference_scipy(inst, seconds: float) -> dict | None:
    """The reference's own run_wrgn (numpy + scipy csr_matvec, one thread per
    trajectory, as solver.py runs each start) on a bounded sample: a k-step
    pursuit (GammaSchedule(0.9, 1.5, k): same per-iteration work).  The WeightedGraph is built
    straight from the instance's CSR (the reference constructor, graph.py:35-46)."""
    mod = reference_module()
    if mod is None:
        return None
    D, RG, where = mod
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    g = RG.WeightedGraph(inst.graph.n, np.array(inst.graph.indptr), np.array(inst.graph.indices),
                         np.array(inst.graph.w, dtype=np.float64))
    # the loop's own rate, as for the port: T(k) - T(2) over k - 2 iterations
    # (run_wrgn's x0 check -- one more SpMV -- and set-up are in both; a linear
    # schedule needs 2 iterations)
    t0 = time.perf_counter()
    D.run_wrgn(g, inst.x0, D.GammaSchedule(0.9, 1.5, 2))
    t1 = time.perf_counter() - t0
    k = int(min(1000, max(4, seconds / max(t1 / 3, 1e-6))))
    t0 = time.perf_counter()
    D.run_wrgn(g, inst.x0, D.GammaSchedule(0.9, 1.5, k))
    tk = time.perf_counter() - t0
    dt = tk - t1
    per_k = k - 2
    if dt <= 0.05 * tk:
        dt, per_k = tk, k
    del g
    return {"value": inst.m * per_k / dt, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"graphnorm.dynamics.run_wrgn (unmodified reference from {where}, scipy csr_matvec), "
                      f"{k}-iteration pursuit on {inst.name}: T({k}) - T(2) = {dt:.2f} s (T(2) = {t1:.2f} s holds "
                      f"the x0 check and set-up)",
            "iters": per_k, "seconds": dt}


def cpu_baselines(inst, seconds: float) -> dict:
    """cpu_baseline for the JSON line: the port on every host thread (the
    reported value), plus the port on one thread and the reference's own
    scipy run_wrgn (one thread per trajectory: what the reference does)."""
    threads = host_threads()
    par = cpu_port(inst, seconds, threads)
    one = cpu_port(inst, seconds / 2, 1)
    ref = None
    try:
        ref = cpu_reference_scipy(inst, seconds / 2)
    except MemoryError:
        ref = None
    out = {k: par[k] for k in ("value", "unit", "cores", "kind", "sample")}
    out["port_1thread"] = {k: one[k] for k in ("value", "cores", "sample")}
    out["reference_scipy"] = ({k: ref[k] for k in ("value", "cores", "kind", "sample")} if ref else
                              {"unavailable": "graphnorm not importable (baseline/_ref missing)"})
    return out


def run_reference(args, ws, rank) -> int:
    """--impl reference: the reference's CPU path on the host cores (rank 0
    only).  Each step times the oracle port of the reference's arithmetic on
    every host thread over a bounded sample of the workload; the reference's
    own scipy run_wrgn and the 1-thread port are reported beside it."""
    if rank != 0:
        return 0
    inst, _ = make_instance(args.config, 0, 1, args.scale)
    threads = host_threads()
    vals, base = [], None
    for i in range(args.warmup + args.steps):
        r = cpu_port(inst, args.ref_seconds, threads)
        if i >= args.warmup:
            vals.append(r["value"])
            base = r
    v = statistics.median(vals)
    extra = cpu_baselines(inst, 2 * args.ref_seconds)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "higher_is_better": True,
        "scaling": "strong" if args.config == "C5" and args.engine == "part" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generators, paper_2605_05330_b200/generators.py)",
        "config": config_dict(args, inst, ws if ws > 1 else args.gpus, engine_dtype(args, inst)),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": base["kind"], "sample": base["sample"],
                         "port_1thread": extra["port_1thread"], "reference_scipy": extra["reference_scipy"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def ncu_traffic(key: str, iters: int):
    """DRAM bytes (read + write) per launch of `iters` iterations, from the
    committed ncu --set full summary of the same kernel (scaled by iterations
    when the capture ran fewer)."""
    f = ROOT / "profiles" / "ncu_summary.json"
    if f.exists():
        try:
            d = json.loads(f.read_text()).get(key, {})
            if d.get("dram_bytes_per_launch") is None:
                return None
            return d["dram_bytes_per_launch"] / (d.get("iters_per_launch") or iters) * iters
        except Exception:
            return None
    return None


def gather_ceiling(key: str, ms_per_iter: float) -> dict | None:
    """The step kernel against the measured gather ceiling: the L1-missing
    sectors one iteration issues (lts__t_sectors_srcunit_tex_op_read from the
    committed ncu capture of the same kernel, profiles/ncu_summary.json) per
    second of this run, over the rate random L1-missing loads reach on this
    GPU (tools/gather_ceiling.cu, profiles/r02_gather_ceiling.jsonl: the
    L2-resident 64 MB table)."""
    try:
        d = json.loads((ROOT / "profiles" / "ncu_summary.json").read_text()).get(key, {})
        sectors = d.get("l2_read_sectors_per_launch") and d["l2_read_sectors_per_launch"] / d.get("iters_per_launch", 1)
        ceil = [json.loads(s) for s in (ROOT / "profiles" / "r02_gather_ceiling.jsonl").read_text().splitlines()]
        ceil = max(c["gloads_per_s"] for c in ceil if c["case"] == "global" and c.get("table_mb") == 64) * 1e9
    except Exception:
        return None
    if not sectors:
        return None
    rate = sectors / (ms_per_iter * 1e-3)
    return {"l2_read_sectors_per_iter": sectors, "sectors_per_s": rate, "ceiling_loads_per_s": ceil,
            "frac": rate / ceil, "source": f"{d.get('label')} (ncu) / tools/gather_ceiling.cu (random 8-byte "
                                          "loads over a 64 MB L2-resident table, 1.0 per SM per cycle)"}


def peak_hbm() -> tuple[float, str]:
    pf = ROOT / "MEASURED_PEAKS.json"
    if pf.exists():
        peaks = json.loads(pf.read_text())
        if "hbm_gbs" in peaks:
            return float(peaks["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_note(traffic, algo, certificates=False):
    if traffic is None:
        return None
    if certificates and traffic < 0.9 * algo:
        return (f"DRAM traffic is {traffic / algo:.2f}x the algorithmic bytes: rows settled by a zero-row certificate "
                "are not walked (roofline.walked_fraction), so most of the adjacency is not read")
    if traffic < 0.5 * algo:
        return (f"DRAM traffic is {traffic / algo:.3f}x the algorithmic bytes: the graph stays in L2/shared memory "
                "across the iterations of a launch, so achieved/frac are the algorithmic rate of SURVEY 8(d), not "
                "DRAM bandwidth")
    return f"DRAM traffic is {traffic / algo:.2f}x the algorithmic bytes (index stream plus L2 misses of the gathers)"


# ---------------------------------------------------------------- GPU arms

def run_partitioned(args, ws, rank, local, inst, torch, P, E, setup_t0) -> int:
    """C5 as BASELINE names it: the graph vertex-range partitioned over the N
    ranks (partition.py), each rank building only its own part from its own
    rows.  Every run: fence the ranks, gn_part_begin, the halo handshake
    (once), then all iterations from one CUDA-graph launch (gn_part_run: with
    N > 1 the graph holds the flag waits, boundary and interior steps, the
    coalesced pushes into the peers' ghost slots and the flags).  --halo nccl
    runs the host-driven pack / NCCL send-recv / unpack loop instead.
    Strong scaling: the graph is the same at every N.  Timed with CUDA events
    on the stream the engine launches on, max over ranks."""
    from paper_2605_05330_b200.partition import (DistExchange, DistPeerExchange, EngineBackend, NoExchange,
                                                 build_partition, run_partition)

    dtype = engine_dtype(args, inst)
    sched = P.GammaSchedule.pursuit(iterations=args.iters)
    gam = sched.table()
    iters = len(gam)
    t_spec = time.perf_counter()
    spec = build_partition(inst.graph, ws, rank)
    be = EngineBackend(spec, dtype=dtype, device=local)
    setup_s = time.perf_counter() - setup_t0
    spec_s = time.perf_counter() - t_spec
    if ws == 1:
        ex = NoExchange(be)
    else:
        ex = DistPeerExchange(be) if args.halo == "peer" else DistExchange(be)
    x0l = spec.local_x0(inst.x0)
    x0_pin = torch.from_numpy(x0l).pin_memory()
    x0p = x0_pin.numpy()
    dev = torch.device("cuda", local)
    devsched = ex.device_schedule

    def timed_run():
        ex.fence()
        be.begin(x0p, gam)
        ex.setup()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if devsched:
            be.run(0, iters)
        else:
            from paper_2605_05330_b200.partition import partitioned_step

            for k in range(iters):
                partitioned_step(be, ex, k)
        e1.record()
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1)

    for _ in range(args.warmup):
        flush_l2(torch, dev)
        timed_run()
    launches0 = E.launch_count()
    times = []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush_l2(torch, dev)
            times.append(timed_run())
    launches = E.launch_count() - launches0
    total_ms = float(sum(times))
    # e2e through the public API: host x0 in (pinned), every iteration, the owned x out
    e2e = []
    res = None
    for i in range(args.warmup + args.steps):
        ex.fence()
        t0 = time.perf_counter()
        res = run_partition(be, ex, x0p, sched)
        torch.cuda.synchronize(dev)
        if os.environ.get("GN_BENCH_VERBOSE"):
            print(f"e2e step {i}: {1e3 * (time.perf_counter() - t0):.1f} ms; " +
                  ", ".join(f"{k} {1e3 * v:.1f} ms" for k, v in be.last_times.items()), file=sys.stderr, flush=True)
        if i >= args.warmup:
            e2e.append(time.perf_counter() - t0)
    e2e_total = sum(e2e)
    # what the zero-row certificates and settled rows leave of the adjacency
    # walk (one counting run, GN_PART_COUNT=1), and the same pursuit with them
    # off (GN_PART_WITNESS=0: every row walks every iteration -- the plain
    # streaming kernel the ncu captures and the gather ceiling describe).
    # Both outside the timed steps; the outputs are bitwise the same.
    walked, off_ms = None, None
    if ws == 1 and not args.no_certificate_report:
        saved = {k: os.environ.get(k) for k in ("GN_PART_COUNT", "GN_PART_WITNESS")}
        try:
            os.environ["GN_PART_COUNT"] = "1"
            timed_run()
            gat = be.gathers(iters)
            be.end(iters)
            walked = float(gat.sum()) / (2.0 * inst.m * iters)
            os.environ["GN_PART_COUNT"] = "0"
            os.environ["GN_PART_WITNESS"] = "0"
            timed_run()
            flush_l2(torch, dev)
            off_ms = timed_run()
            x_off = be.end(iters)[0]
            if res is not None and not np.array_equal(x_off, res.x):
                raise RuntimeError("certificates changed the result: bench aborted")
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    t = torch.tensor([total_ms, e2e_total, setup_s], device=dev, dtype=torch.float64)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    total_ms, e2e_total, setup_max = (float(v) for v in t.tolist())
    if rank == 0:
        m, n = inst.m, inst.graph.n
        value = m * iters * args.steps / (total_ms * 1e-3)
        peak, peak_src = peak_hbm()
        s_bytes = 8 if dtype == "fp64" else 4
        b_iter = algorithmic_bytes(n, 2 * m, s_bytes)
        achieved = b_iter * iters * args.steps / (total_ms * 1e-3) / 1e9
        traffic = ncu_traffic("C5part", 1) if ws == 1 else None  # per step launch = one iteration
        clk = clocks.summary()
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            cpu = cpu_baselines(inst, args.ref_seconds)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": {"fp64": "f64", "fp32": "f32-gather/f64-state", "fp32_pure": "f32"}[dtype],
            "data": "synthetic (seeded generators, paper_2605_05330_b200/generators.py)",
            "config": config_dict(args, inst, ws, dtype),
            "partition": {"ghosts_rank0": spec.n_ghost, "owned_rank0": spec.n_own,
                          "host_setup_s_rank0": round(setup_s, 2), "host_setup_s_max": round(setup_max, 2),
                          "part_build_s_rank0": round(spec_s, 2)},
            "e2e": {"value": m * iters * args.steps / e2e_total, "unit": UNIT,
                    "h2d_bytes_per_step": 8 * (spec.n_own + spec.n_ghost) + 8 * iters,
                    "d2h_bytes_per_step": 8 * spec.n_own + 32 * iters,
                    "api": "partition.run_partition (host x0 in, owned x and per-iteration stats out), rank 0 shown"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * ws, "unit": "GB/s",
                         "frac": achieved / (peak * ws), "traffic": traffic,
                         "traffic_per": "iteration: mean DRAM bytes of one iteration's launches over the whole pursuit "
                                        "(ncu metrics sweep of every k_part_* launch, profiles/r02_c5s24_pursuit_sweep.json)",
                         "traffic_note": traffic_note(traffic, b_iter, certificates=True),
                         "kernel": "gn::k_part_step (1 launch per iteration per part, replayed from a CUDA graph)" + (
                             "" if ws == 1 else (" + coalesced pushes into the peers' ghost slots (CUDA IPC)"
                                                 if args.halo == "peer" else " + NCCL halo")),
                         "b_iter": b_iter, "peak_source": peak_src + (f" x {ws} GPUs" if ws > 1 else ""),
                         "achieved_over": "the whole iteration (step + long-row combine launches)",
                         "achieved_note": "algorithmic bytes of every iteration over the measured time; rows the "
                                          "zero-row certificates settle are not walked (walked_fraction), so this is a "
                                          "rate of work done or proven unnecessary, not of bytes moved; "
                                          "certificates_off is the same pursuit with every row walked",
                         "walked_fraction": walked,
                         "certificates_off": None if off_ms is None else {
                             "ms_per_step": off_ms, "value": m * iters / (off_ms * 1e-3),
                             "achieved": b_iter * iters / (off_ms * 1e-3) / 1e9,
                             "frac": b_iter * iters / (off_ms * 1e-3) / 1e9 / peak,
                             "traffic": ncu_traffic("C5part_plain", 1),
                             "gather_ceiling": gather_ceiling("C5part_plain", off_ms / iters) if dtype == "fp64" else None,
                             "result": "bitwise equal to the timed runs' x"}},
            "cpu_baseline": cpu,
            "clocks": {k: clk[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
            "gpu_launches": int(launches),
        }
        print(json.dumps(line), flush=True)
    if hasattr(ex, "close"):
        ex.fence()  # no peer still writes into our buffers
        ex.close()
    be.close()
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def run_single(args, ws, rank, local, inst, batch, torch, P, E) -> int:
    """C1-C4 (and C5 --engine loop): one engine call per step on each rank
    (replicas, or the rank's own batch shard for C4)."""
    from paper_2605_05330_b200.batch import GraphBatch

    dev = torch.device("cuda", local)
    g = inst.graph
    dtype = engine_dtype(args, inst)
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
            # per-graph traces (step_inf, fallbacks, objective) are part of every run (dynamics.py:165-168)
            r = gb.run(None, sched, device_x0=x0_dev.data_ptr(), device_x_out=x_out.data_ptr(), traces=True)
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
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush_l2(torch, dev)
            torch.cuda.synchronize()
            st = device_step()
            step_ms.append(st.total_ms)
            loop_ms.append(st.loop_ms)
    barrier()
    launches = E.launch_count() - launches0
    total_ms = float(sum(step_ms))
    if ws > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    edges_all = inst.m * ws * starts
    value = edges_all * iters * args.steps / (total_ms * 1e-3)

    # ---- e2e through the public API: host x0 in, MIS out, every step; the
    # state stays in HBM between the run and the rounding (device_state).
    # The harness has torch loaded (millions of tracked objects): move them
    # out of the collector's way so a full collection cannot land in a step.
    gc.collect()
    gc.freeze()
    x0_host = torch.from_numpy(np.ascontiguousarray(inst.x0)).pin_memory().numpy()
    x0s_host = torch.from_numpy(np.ascontiguousarray(x0s)).pin_memory().numpy()
    e2e_t, round_t = [], []
    h2d = d2h = 0
    for i in range(args.warmup + args.steps):
        barrier()
        t0 = time.perf_counter()
        if batch is not None:
            r = gb.run(x0_host, sched)
            t1 = time.perf_counter()
            sol = P.round_to_mis(g, r.x)  # the packed graph: per-graph roundings, block by block
            xbytes = 8 * g.n
        elif starts > 1:
            r = P.run_multi(g, x0s_host, sched, dtype=dtype, device=local)
            t1 = time.perf_counter()
            sol = P.round_many(g, r.x)
            xbytes = 8 * g.n * starts
        else:
            r = P.run_engine(g, x0_host, sched, dtype=dtype, device=local, device_state=True)
            t1 = time.perf_counter()
            sol = P.round_to_mis(g, r.x)
            xbytes = 8 * g.n  # x0 uploaded by run_engine; x is handed to the rounding in HBM
        barrier()
        if os.environ.get("GN_BENCH_VERBOSE"):
            print(f"e2e step {i}: run {1e3 * (t1 - t0):.2f} ms, round {1e3 * (time.perf_counter() - t1):.2f} ms, "
                  f"call {r.stats['total_ms']:.2f} ms loop {r.stats['loop_ms']:.2f} ms", file=sys.stderr, flush=True)
        if i >= args.warmup:
            e2e_t.append(time.perf_counter() - t0)
            round_t.append(time.perf_counter() - t1)
            h2d = r.stats["h2d_bytes"] + xbytes  # + the rounding's state upload, or run_engine's x0 upload
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

    peak, peak_src = peak_hbm()
    s_bytes = 8 if dtype == "fp64" else 4  # s = element size of the state vectors
    # SURVEY 8(d) per iteration; with several starts the index stream is read
    # once for all of them and the state streams once per start
    b_iter = algorithmic_bytes(g.n, 2 * inst.m, s_bytes) + 3 * s_bytes * g.n * (starts - 1)
    loop_avg = statistics.mean(loop_ms)
    achieved = b_iter * iters / (loop_avg * 1e-3) / 1e9
    traffic = ncu_traffic(args.config, iters) if starts == 1 else None
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baselines(inst, args.ref_seconds)
    clk = clocks.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": {"fp64": "f64", "fp32": "f32-gather/f64-state", "fp32_pure": "f32"}[dtype],
        "data": "synthetic (seeded generators, paper_2605_05330_b200/generators.py)",
        "config": config_dict(args, inst, ws, dtype),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "api": ("paper_2605_05330_b200.run_multi + round_many" if starts > 1 else
                        "GraphBatch.run + round_to_mis" if batch is not None else
                        "paper_2605_05330_b200.run_engine(device_state=True) + round_to_mis") +
                       " (host numpy in, MIS out)",
                "round_ms_per_step": 1e3 * statistics.mean(round_t) if round_t else None},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "kernel": kernel_name,
                     "bytes_per_launch": b_iter * iters, "b_iter": b_iter, "peak_source": peak_src,
                     "loop_ms": loop_avg, "traffic_note": traffic_note(traffic, b_iter * iters)},
        "cpu_baseline": cpu,
        "clocks": {k: clk[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
        "gpu_launches": int(launches),
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--engine", default="part", choices=["part", "loop"],
                    help="C5: the partitioned engine (default; one part per GPU) or the single-GPU loop kernel")
    ap.add_argument("--scale", type=int, default=24, help="R-MAT scale for C5 (BASELINE: 24)")
    ap.add_argument("--dtype", default=None, help="engine dtype (default: fp64 for C1-C3, fp32 for C4/C5)")
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--ref-seconds", type=float, default=6.0)
    ap.add_argument("--no-certificate-report", action="store_true",
                    help="C5: skip the counting run and the certificates-off run after the timed steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--halo", choices=["peer", "nccl"], default="peer",
                    help="C5 with N > 1: coalesced pushes into the peers' ghost slots (default) or NCCL send/recv")
    ap.add_argument("--partition", action="store_true", help="(kept for old command lines: same as --engine part)")
    ap.add_argument("--starts", type=int, default=1,
                    help="starts per instance (SURVEY 8f f1): >1 runs them together through gn_multi_run")
    ap.add_argument("--dry-run", action="store_true", help=argparse.SUPPRESS)  # rank env check (tests)
    args = ap.parse_args()
    if args.partition:
        args.engine = "part"
    ws, rank, local = dist_env()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.dry_run:
        print(json.dumps({"rank": rank, "world_size": ws, "local_rank": local, "gpus": args.gpus,
                          "master": os.environ.get("MASTER_ADDR"), "config": args.config}), flush=True)
        return 0
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
    setup_t0 = time.perf_counter()
    inst, batch = make_instance(args.config, rank, ws, args.scale)
    if args.config == "C5" and args.engine == "part":
        return run_partitioned(args, ws, rank, local, inst, torch, P, E, setup_t0)
    return run_single(args, ws, rank, local, inst, batch, torch, P, E)


if __name__ == "__main__":
    sys.exit(main())
