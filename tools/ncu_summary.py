"""Summarise an ncu report (--set full) or a launch list into profiles/.

    python tools/ncu_summary.py rep  gpurun_out/prof_c2.ncu-rep  --label r01_c2 [--config C2] [--iters 1000]
    python tools/ncu_summary.py launches gpurun_out/launches.csv --label r01_bench_launches
"""
import argparse
import csv
import io
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "smsp__inst_executed.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
    "l1tex__t_sector_hit_rate.pct", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__warps_launched.sum",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = dict(zip(hdr, v))
        u = dict(zip(hdr, units))
        res.append((d, u))
    return res


def num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def summarize_rep(rep, label, config, iters, names=None):
    out = {}
    for idx, (d, u) in enumerate(raw(rep)):
        name = d.get("Kernel Name", "?")
        if names is not None:  # one entry per launch, labelled
            name = f"{idx}: {names[idx] if idx < len(names) else '?'}: {name.split('(')[0]}"
        m = {}
        for k in KEYS:
            if k in d:
                val = num(d[k])
                unit = u.get(k, "")
                if val is not None and unit in SCALE:
                    val *= SCALE[unit]
                    unit = "B" if "byte" in unit else ("s" if "second" in unit else unit)
                m[k] = {"value": val, "unit": unit}
        stalls = {k.split("stalled_")[1].split("_per")[0]: num(d[k]) for k in d
                  if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")}
        m["top_stalls_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -(kv[1] or 0))[:6])
        dram = (m.get("dram__bytes_read.sum", {}).get("value") or 0) + (m.get("dram__bytes_write.sum", {}).get("value") or 0)
        m["dram_bytes_per_launch"] = dram
        if iters:
            m["dram_bytes_per_iteration"] = dram / iters
        out[name] = m
    path = ROOT / "profiles" / f"{label}.json"
    path.write_text(json.dumps({"report": Path(rep).name, "config": config, "iters_per_launch": iters,
                                "kernels": out}, indent=1))
    if config:
        sf = ROOT / "profiles" / "ncu_summary.json"
        s = json.loads(sf.read_text()) if sf.exists() else {}
        loop = [m for n, m in out.items()
                if any(k in n for k in ("k_gn_loop", "k_gn_batch", "k_gn_multi", "k_part_step"))]
        if loop:
            s[config] = {"label": label, "dram_bytes_per_launch": loop[0]["dram_bytes_per_launch"],
                         "l2_read_sectors_per_launch":
                             loop[0].get("lts__t_sectors_srcunit_tex_op_read.sum", {}).get("value"),
                         "iters_per_launch": iters}
            sf.write_text(json.dumps(s, indent=1))
    print(path)


def summarize_launches(csvfile, label):
    rows = [r for r in csv.reader(open(csvfile)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ci = {h: i for i, h in enumerate(hdr)}
    tot = {}
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        name = r[ci["Kernel Name"]]
        v = num(r[ci["Metric Value"]])
        unit = r[ci["Metric Unit"]]
        v = v * SCALE.get(unit, 1e-9)
        t = tot.setdefault(name, [0, 0.0])
        t[0] += 1
        t[1] += v
    total = sum(t[1] for t in tot.values())
    lines = [f"# {label}: ncu launch list (gpu__time_duration.sum, --clock-control none; cold, serialised)",
             "", "| share | launches | total ms | kernel |", "|---:|---:|---:|---|"]
    for name, (c, s) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {s / total * 100:.2f}% | {c} | {s * 1e3:.3f} | `{name[:110]}` |")
    path = ROOT / "profiles" / f"{label}.md"
    path.write_text("\n".join(lines) + "\n")
    print(path)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("kind", choices=["rep", "launches"])
    ap.add_argument("path")
    ap.add_argument("--label", required=True)
    ap.add_argument("--config")
    ap.add_argument("--iters", type=int)
    ap.add_argument("--names", help="comma-separated labels, one per launch (one entry per launch)")
    a = ap.parse_args()
    if a.kind == "rep":
        summarize_rep(a.path, a.label, a.config, a.iters, a.names.split(",") if a.names else None)
    else:
        summarize_launches(a.path, a.label)
