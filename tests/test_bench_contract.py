"""bench.py's JSON-line contract on the CPU-only arm (the reference arm times the
reference in baseline/_ref, else the oracle port; the GPU arm runs on a B200)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--workload", "ses_c1", "--steps", "1", "--warmup", "1",
                          "--cpu-seconds", "0.5"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is False
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    # the time-to-eps uses the reference's own recorded iteration count (long.json, C1)
    assert d["config"]["reference_iterations"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_more_gpus_than_visible_fails_loudly():
    """--gpus N outside torchrun spawns N ranks, and refuses when fewer devices are visible
    (round 1 silently ran one rank and reported n_gpus 1)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--workload", "ses_c1", "--steps", "1", "--warmup", "1",
                          "--no-cpu-baseline"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT)
    import torch
    if torch.cuda.device_count() >= 2:
        return
    assert out.returncode != 0 and "visible" in out.stdout + out.stderr


def test_reference_counts_come_from_reference_records():
    """The CPU arm's iteration count is the reference's own recorded count for the
    workload's family (largest recorded n), never a device count."""
    sys.path.insert(0, ROOT)
    import bench
    its, n, threads = bench.reference_counts(bench.WORKLOADS["ses_c4"])
    rec = json.load(open(os.path.join(ROOT, "tests", "golden", "headline",
                                      f"ses_n{n}_t1.json")))
    assert its == rec["solve"]["iterations"] and n >= 100000 and 1 in threads
    its, n, _ = bench.reference_counts(bench.WORKLOADS["svm_c3"])
    assert n >= 10000 and its > 0
    its, n, _ = bench.reference_counts(bench.WORKLOADS["ses_c1"])
    assert (its, n) == (82518, 10000)     # long.json, threads=1
