"""CPU: the bench.py reference arm prints the driver's JSON contract line
(the oracle port timed on the host cores; no GPU involved)."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "1", "--warmup", "3", "--ref-seconds", "0.2"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling", "dtype",
                "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert cb["cores"] == len(__import__("os").sched_getaffinity(0))
    assert cb["port_1thread"]["cores"] == 1
    ref = cb["reference_scipy"]
    assert ref.get("kind") == "reference" and ref["cores"] == 1 and ref["value"] > 0, ref
    # same config dict as the GPU arm prints (the driver compares them)
    assert set(line["config"]) >= {"workload", "n", "m", "iters", "schedule", "parallelism", "engine",
                                   "engine_dtype", "starts", "l2", "index_format", "inputs"}


def test_gpus_n_spawns_one_rank_per_gpu():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks with
    the torchrun environment (the driver's SCALE command line)."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world_size"] == 2 and d["local_rank"] == d["rank"] and d["master"] == "127.0.0.1" for d in lines)
