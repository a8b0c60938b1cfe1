"""Pin the CPU restatement of paper Algorithm 3 (oracle_fast_osbf,
filters2d.hpp:105-154) before trusting it: golden outputs of the unmodified
reference, the reference's own known answers (test_filters2d.cpp:169-186),
and bit-exact agreement with the compiled reference on fresh inputs."""
import os

import numpy as np
import pytest

import oracle
from conftest import bits, fastosbf_golden_cases, load_golden


@pytest.mark.parametrize("path", fastosbf_golden_cases(), ids=os.path.basename)
def test_fast_osbf_oracle_matches_golden(oracle_lib, path):
    g = load_golden(path)
    x, r, it = g["input"].astype(np.float64), int(g["radius"]), int(g["iterations"])
    got = (np.stack([oracle_lib.fast_osbf(c, r, it) for c in x]) if x.ndim == 3
           else oracle_lib.fast_osbf(x, r, it))
    assert np.array_equal(bits(got), bits(g["output"]))


def test_fast_osbf_known_answers(oracle_lib):
    # test_filters2d.cpp:169-177: constant planes and ideal steps are fixed points
    c = np.full((9, 9), 11.0)
    assert np.array_equal(oracle_lib.fast_osbf(c, 3, 2), c)
    x = np.arange(32)[None, :].repeat(16, 0)
    step = np.where(x < 16, 0.0, 100.0)
    for r in (1, 2, 5):
        assert np.array_equal(oracle_lib.fast_osbf(step, r, 1), step)
    # filters2d.hpp:107-110: radius checked before iterations, even for 0 iterations
    for r, it in ((0, 0), (0, 1), (1, -1)):
        with pytest.raises(oracle.CheckerError):
            oracle_lib.fast_osbf(c, r, it)
    assert np.array_equal(oracle_lib.fast_osbf(c, 1, 0), c)


def test_fast_osbf_tracks_exact(oracle_lib):
    # test_filters2d.cpp:179-186: RMSE(exact, fast) <= 5 on a structured image
    from paper_2108_05021_b200 import synth

    p = synth.make_input("C1", shrink=4)[0].astype(np.float64) * 255.0
    for r in (2, 6):
        e, f = oracle_lib.osbf(p, r, 10), oracle_lib.fast_osbf(p, r, 10)
        assert float(np.sqrt(np.mean((e - f) ** 2))) <= 5.0


@pytest.mark.parametrize("seed", range(3))
def test_fast_osbf_oracle_matches_compiled_reference(oracle_lib, reference_lib, seed):
    rng = np.random.default_rng(500 + seed)
    for _ in range(4):
        h, w = int(rng.integers(1, 60)), int(rng.integers(1, 60))
        r = int(rng.choice([1, 2, 3, 5, 9, 16]))
        p = rng.random((h, w)) * 255
        assert np.array_equal(bits(oracle_lib.fast_osbf(p, r, 3)),
                              bits(reference_lib.fast_osbf(p, r, 3)))
