"""box_filter (filters2d.hpp:38-56): the oracle
restatement pinned to the reference (golden outputs of the unmodified
reference, known answers, the compiled reference), and the GPU path
(osbf_gpu_box_filter) bit-identical to it."""
import os

import numpy as np
import pytest

import oracle
from conftest import bits, boxfilter_golden_cases, load_golden


@pytest.mark.parametrize("path", boxfilter_golden_cases(), ids=os.path.basename)
def test_box_oracle_matches_golden(oracle_lib, path):
    g = load_golden(path)
    x, r, it = g["input"].astype(np.float64), int(g["radius"]), int(g["iterations"])
    got = (np.stack([oracle_lib.box_filter(c, r, it) for c in x]) if x.ndim == 3
           else oracle_lib.box_filter(x, r, it))
    assert np.array_equal(bits(got), bits(g["output"]))


def test_box_oracle_known_answers(oracle_lib):
    c = np.full((7, 9), 5.0)
    for r in (1, 2, 6):
        assert np.array_equal(oracle_lib.box_filter(c, r, 4), c)  # test_filters2d.cpp:44-48
    for r, it in ((0, 0), (0, 1), (1, -1)):
        with pytest.raises(oracle.CheckerError):
            oracle_lib.box_filter(c, r, it)


def test_box_oracle_matches_compiled_reference(oracle_lib, reference_lib):
    rng = np.random.default_rng(61)
    for _ in range(6):
        h, w = int(rng.integers(1, 50)), int(rng.integers(1, 50))
        r = int(rng.choice([1, 2, 5, 11]))
        p = rng.random((h, w)) * 100 - 50
        assert np.array_equal(bits(oracle_lib.box_filter(p, r, 3)),
                              bits(reference_lib.box_filter(p, r, 3)))


@pytest.mark.gpu
@pytest.mark.parametrize("path", boxfilter_golden_cases(), ids=os.path.basename)
def test_box_gpu_matches_reference_golden(ctx, path):
    import torch

    import paper_2108_05021_b200 as ob

    g = load_golden(path)
    x, r, it = g["input"], int(g["radius"]), int(g["iterations"])
    if x.ndim == 3:
        cfg = ob.FilterConfig(radius=r, iterations=it, variant=ob.FilterVariant.Box)
        host = np.stack(ob.filter_multichannel([c.astype(np.float64) for c in x], cfg))
        assert np.array_equal(bits(host), bits(g["output"]))
    got = ctx.box_filter(torch.from_numpy(np.ascontiguousarray(x)).cuda(), r, it).cpu().numpy()
    assert np.array_equal(bits(got), bits(g["output"]))
    assert np.array_equal(bits(ctx.box_filter_host(x, r, it)), bits(g["output"]))


@pytest.mark.gpu
def test_box_gpu_random_and_errors(ctx, oracle_lib):
    import torch

    import paper_2108_05021_b200 as ob

    rng = np.random.default_rng(62)
    for _ in range(4):
        h, w = int(rng.integers(1, 500)), int(rng.integers(1, 500))
        r = int(rng.choice([1, 3, 8, 30]))
        p = rng.random((h, w)) * 255
        got = ctx.box_filter(torch.from_numpy(p).cuda(), r, 2).cpu().numpy()
        assert np.array_equal(bits(got), bits(oracle_lib.box_filter(p, r, 2)))
    for r, it in ((0, 0), (0, 2), (2, -1)):
        with pytest.raises(ob.InvalidArgument):
            ob.box_filter(np.ones((4, 4)), r, it)
