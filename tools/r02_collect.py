"""Collect the outputs of tools/r02_final2.sh (gpurun_out/<dir>) into
profiles/: bench lines, ncu summaries of the C5 step at three stages of the
pursuit and with the certificates off, the per-launch metrics sweep of one
whole pursuit (L2 read sectors, DRAM bytes and time per iteration), the
launch list, the A/B and active-row probes.  Updates profiles/ncu_summary.json
(C5part: DRAM bytes per iteration averaged over the pursuit; C5part_plain:
the plain kernel's sectors and DRAM bytes per iteration).

    python tools/r02_collect.py gpurun_out/r2f2
"""
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"


def num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def sweep(csvfile: Path, out: Path, iters: int = 1000) -> dict:
    """ncu --metrics sweep over every k_part_* launch of one pursuit."""
    rows = [r for r in csv.reader(open(csvfile)) if r and r[0] and not r[0].startswith("==")]
    hdr = rows[0]
    ci = {h: i for i, h in enumerate(hdr)}
    per = {}  # launch id -> {kernel, metric: value}
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        d = per.setdefault(int(r[ci["ID"]]), {"kernel": r[ci["Kernel Name"]].split("(")[0].split("<")[0].split("::")[-1].replace("void ", "").strip()})
        v, unit = num(r[ci["Metric Value"]]), r[ci["Metric Unit"]]
        scale = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                 "sector": 1}.get(unit, 1)
        d[r[ci["Metric Name"]]] = v * scale
    kinds = {}
    for _, d in sorted(per.items()):
        kinds.setdefault(d["kernel"], []).append(d)
    steps = kinds.get("k_part_step", [])
    n = len(steps)
    res = {"iterations": n, "kernels": {}, "note": "ncu per-launch values (cold cache, serialised): sectors and bytes "
           "are exact per launch, times are not the graph-replayed times"}
    tot = {"sectors": 0.0, "dram": 0.0, "time": 0.0}
    for k, lst in kinds.items():
        sec = [d.get("lts__t_sectors_srcunit_tex_op_read.sum", 0.0) for d in lst]
        dram = [d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0) for d in lst]
        t = [d.get("gpu__time_duration.sum", 0.0) for d in lst]
        tot["sectors"] += sum(sec)
        tot["dram"] += sum(dram)
        tot["time"] += sum(t)
        res["kernels"][k] = {
            "launches": len(lst), "l2_read_sectors_total": sum(sec), "dram_bytes_total": sum(dram),
            "time_s_total": sum(t),
            "l2_read_sectors_by_100": [round(sum(sec[j:j + 100]) / max(len(sec[j:j + 100]), 1)) for j in range(0, len(sec), 100)],
            "dram_bytes_by_100": [round(sum(dram[j:j + 100]) / max(len(dram[j:j + 100]), 1)) for j in range(0, len(dram), 100)],
            "time_us_by_100": [round(1e6 * sum(t[j:j + 100]) / max(len(t[j:j + 100]), 1), 1) for j in range(0, len(t), 100)],
        }
    res["per_iteration_mean"] = {"l2_read_sectors": tot["sectors"] / max(n, 1), "dram_bytes": tot["dram"] / max(n, 1),
                                 "ncu_time_us": 1e6 * tot["time"] / max(n, 1)}
    out.write_text(json.dumps(res, indent=1))
    return res


def main():
    src = Path(sys.argv[1])
    for a, b in (("bench_c5.json", "r02_bench_c5.json"), ("bench_c5_fp32.json", "r02_bench_c5_fp32.json"),
                 ("bench_C2.json", "r02_bench_c2.json"), ("bench_C3.json", "r02_bench_c3.json"),
                 ("bench_C4.json", "r02_bench_c4.json"), ("bench_ref.json", "r02_bench_c5_reference.json"),
                 ("witness_ab.jsonl", "r02_c5s24_certificates_ab.jsonl"), ("active.json", "r02_c5s24_active_rows.json")):
        if (src / a).exists() and (src / a).stat().st_size:
            shutil.copy(src / a, PROF / b)
            print(PROF / b)
    if (src / "fp32_excursions").is_dir():
        for f in (src / "fp32_excursions").glob("*.json"):
            shutil.copy(f, PROF / "r02_fp32_excursions" / f.name)
    for rep, label, cfg in (("c5step_k5.ncu-rep", "r02_c5s24_step_cert_k5_ncu", None),
                            ("c5step_k300.ncu-rep", "r02_c5s24_step_cert_k300_ncu", None),
                            ("c5step_k900.ncu-rep", "r02_c5s24_step_cert_k900_ncu", None),
                            ("c5step_plain.ncu-rep", "r02_c5s24_step_plain_spw16_ncu", "C5part_plain")):
        if (src / rep).exists():
            cmd = [sys.executable, str(ROOT / "tools" / "ncu_summary.py"), "rep", str(src / rep), "--label", label,
                   "--iters", "1"]
            if cfg:
                cmd += ["--config", cfg]
            subprocess.run(cmd, check=True)
    if (src / "sweep.csv").exists():
        r = sweep(src / "sweep.csv", PROF / "r02_c5s24_pursuit_sweep.json")
        sf = PROF / "ncu_summary.json"
        s = json.loads(sf.read_text())
        s["C5part"] = {"label": "r02_c5s24_pursuit_sweep (every k_part_* launch of one 1000-iteration pursuit; mean per "
                                "iteration)",
                       "dram_bytes_per_launch": r["per_iteration_mean"]["dram_bytes"],
                       "l2_read_sectors_per_launch": r["per_iteration_mean"]["l2_read_sectors"], "iters_per_launch": 1}
        sf.write_text(json.dumps(s, indent=1))
        print(PROF / "r02_c5s24_pursuit_sweep.json", r["per_iteration_mean"])
    if (src / "launches.csv").exists():
        subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), "launches", str(src / "launches.csv"),
                        "--label", "r02_bench_c5_launches"], check=True)


if __name__ == "__main__":
    main()
