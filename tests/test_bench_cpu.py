"""The driver's bench.py contract, checked without a GPU: defaults (N=1,
W >= 3 warm-up steps, a K that finishes in minutes), the reference arm, and
the JSON keys the driver reads are produced by the code paths (by name)."""
import os
import subprocess
import sys


ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_bench_defaults(monkeypatch):
    sys.path.insert(0, ROOT)
    import bench

    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse()
    assert a.gpus == 1 and a.warmup >= 3 and 1 <= a.steps <= 100
    assert a.impl == "ours" and a.workload == "C5" and a.mode == "fast"
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--gpus", "2"])
    a = bench.parse()
    assert a.impl == "reference" and a.gpus == 2


def test_bench_json_keys_present_in_source():
    src = open(os.path.join(ROOT, "bench.py")).read()
    for key in ('"metric"', '"value"', '"unit"', '"n_gpus"', '"steps"', '"warmup"',
                '"ms_per_step"', '"higher_is_better"', '"scaling"', '"vs_baseline"', '"dtype"',
                '"data"', '"config"', '"roofline"', '"cpu_baseline"', '"e2e"',
                '"gpu_launches"', '"clocks"', '"impl"', '"h2d_bytes_per_step"',
                '"d2h_bytes_per_step"'):
        assert key in src, key


def test_bench_help_runs_without_gpu():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "--workload" in r.stdout
