"""Pin the CPU oracle (oracle/osbf_oracle.c) before trusting it.

1. Known-answer tests restated from the reference's own suite.
2. Bit-exact agreement with the committed golden fixtures (outputs of the
   unmodified reference, tests/golden/make_golden.py).
3. Bit-exact agreement with the compiled reference (oracle/_ref) on fresh
   seeded inputs, when that library is present.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR, bits, golden_cases, load_golden


def test_sub_windows_table(oracle_lib):
    # core.hpp:212-225 and test_core.cpp:95-114
    r = 3
    wins = oracle_lib.sub_windows(r)
    assert [w[0] for w in wins] == list(range(1, 9))
    for i, (wid, u0, u1, v0, v1) in enumerate(wins):
        assert u0 <= 0 <= u1 and v0 <= 0 <= v1
        pixels = (u1 - u0 + 1) * (v1 - v0 + 1)
        assert pixels == ((r + 1) ** 2 if i < 4 else (r + 1) * (2 * r + 1))
    with pytest.raises(Exception):
        oracle_lib.sub_windows(0)


def test_sat_known_answer(oracle_lib):
    # test_integral.cpp:19-29
    c = oracle_lib.sat(np.array([[1.0, 2.0], [3.0, 4.0]]))
    assert c[0, 0] == 0 and c[0, 2] == 0 and c[2, 0] == 0
    assert (c[1, 1], c[1, 2], c[2, 1], c[2, 2]) == (1.0, 3.0, 4.0, 10.0)
    g = np.load(os.path.join(GOLDEN_DIR, "sat_2x2.npz"))
    assert np.array_equal(bits(c), bits(g["cumsum"]))


def test_rect_mean_known_answers(oracle_lib):
    # test_integral.cpp:42-47, 80-89
    c = oracle_lib.sat(np.ones((5, 5)))
    assert oracle_lib.lib.oracle_rect_sum(c.ctypes.data_as(oracle_lib_dp()), 5, 5, 1, 1, 3, 3) == 9.0
    c = oracle_lib.sat(np.full((4, 6), 3.25))
    assert oracle_lib.rect_mean(c, 6, 4, 0, 0, 5, 3) == 3.25
    assert oracle_lib.rect_mean(c, 6, 4, -3, -3, 2, 2) == 3.25
    tiny = oracle_lib.sat(np.array([[0.0, 100.0]]))
    assert oracle_lib.rect_mean(tiny, 2, 1, 0, 0, 1, 0) == 50.0
    import oracle

    with pytest.raises(oracle.CheckerError) as e:
        oracle_lib.rect_mean(c, 6, 4, 10, 10, 12, 12)
    assert e.value.status == 2  # std::domain_error


def oracle_lib_dp():
    import ctypes

    return ctypes.POINTER(ctypes.c_double)


def test_subwindow_means_known_answers(oracle_lib):
    # test_filters2d.cpp:72-88
    p = np.full((10, 10), 7.25)
    m = oracle_lib.subwindow_means(oracle_lib.sat(p), 10, 10, 4, 5, 2)
    assert np.all(m == 7.25)
    edge = 8
    step = np.where(np.arange(16)[None, :] < edge, 0.0, 100.0).repeat(16, 0)
    c = oracle_lib.sat(step)
    for r in (1, 2, 3):
        assert oracle_lib.subwindow_means(c, 16, 16, edge - 1, 8, r)[4] == 0.0


def test_fixed_points(oracle_lib):
    # test_filters2d.cpp:104-140
    p = np.full((9, 9), 3.5)
    assert np.array_equal(oracle_lib.osbf_step(p, 2), p)
    step = np.where(np.arange(32)[None, :] < 16, 0.0, 100.0).repeat(16, 0)
    for r in (1, 2, 5, 8):
        assert np.array_equal(oracle_lib.osbf_step(step, r), step)
    step64 = np.where(np.arange(64)[None, :] < 32, 0.0, 100.0).repeat(32, 0)
    assert np.array_equal(oracle_lib.osbf(step64, 2, 30), step64)
    rnd = np.random.default_rng(3).random((10, 10))
    assert np.array_equal(oracle_lib.osbf(rnd, 2, 0), rnd)
    # r < 1 with zero iterations is NOT an error (filters2d.hpp:94-97)
    assert np.array_equal(oracle_lib.osbf(rnd, 0, 0), rnd)


@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_matches_golden(oracle_lib, path):
    g = load_golden(path)
    inp, r, it = g["input"].astype(np.float64), int(g["radius"]), int(g["iterations"])
    planes = inp if inp.ndim == 3 else inp[None]
    outs = g["output"] if inp.ndim == 3 else g["output"][None]
    for p, want in zip(planes, outs):
        got = oracle_lib.osbf(p, r, it)
        assert np.array_equal(bits(got), bits(want)), "oracle differs from the reference"
    if it > 0:
        _, sel = oracle_lib.osbf_step(planes[0], r, with_selection=True)
        assert np.array_equal(sel, g["step1_sel"])


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_oracle_matches_compiled_reference(oracle_lib, reference_lib, seed):
    rng = np.random.default_rng(seed)
    h, w = int(rng.integers(1, 70)), int(rng.integers(1, 70))
    for r in (1, 2, 3, 7):
        p = rng.random((h, w)) * 255.0
        assert np.array_equal(bits(oracle_lib.osbf(p, r, 4)), bits(reference_lib.osbf(p, r, 4)))
        u8 = rng.integers(0, 256, (h, w)).astype(np.float64)
        assert np.array_equal(bits(oracle_lib.osbf(u8, r, 6)), bits(reference_lib.osbf(u8, r, 6)))


def test_oracle_thread_count_invariance(oracle_lib):
    # test_filters2d.cpp:374-385
    p = np.random.default_rng(123).random((29, 33)) * 255
    assert np.array_equal(bits(oracle_lib.osbf(p, 2, 2, threads=1)),
                          bits(oracle_lib.osbf(p, 2, 2, threads=4)))
