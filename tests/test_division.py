"""The exact mode's 3-op division by an integer count (osbf_exact2_kernel.cuh
div_by_count) restated in C and compared with IEEE division on the CPU."""
import os
import subprocess

from conftest import ROOT


def test_fma_division_matches_ieee(tmp_path):
    exe = str(tmp_path / "divcheck")
    src = os.path.join(ROOT, "tools", "probes", "divcheck.c")
    subprocess.run(["gcc", "-O2", "-mfma", "-o", exe, src, "-lm"], check=True)
    # exhaustive over integer sums of uint8 windows for counts <= 64, plus
    # random and adversarial doubles (the full 600-count sweep runs in ~40 s)
    res = subprocess.run([exe, "64"], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout
    assert "mismatches 0" in res.stdout
