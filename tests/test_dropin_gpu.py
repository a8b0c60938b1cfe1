"""Run the C++ drop-in test (tests/cpp/test_dropin.cpp) on the GPU: the
reference's hot-path test cases written against include/osbf/*.hpp."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_dropin_suite():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    res = subprocess.run([os.path.join(ROOT, "tests", "cpp", "test_dropin")], capture_output=True,
                         text=True, timeout=600)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "0 failure(s)" in res.stdout
