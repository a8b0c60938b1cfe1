"""3-D extension (filters3d.hpp:55-114): the oracle
restatement pinned to the reference, and osbf_gpu_osbf_3d /
osbf_gpu_box_filter_3d bit-identical to it."""
import os

import numpy as np
import pytest

import oracle
from conftest import bits, filter3d_golden_cases, load_golden


@pytest.mark.parametrize("path", filter3d_golden_cases(), ids=os.path.basename)
def test_3d_oracle_matches_golden(oracle_lib, path):
    g = load_golden(path)
    v, r, it = g["input"], int(g["radius"]), int(g["iterations"])
    f = oracle_lib.osbf_3d if bool(g["osbf3"]) else oracle_lib.box_filter_3d
    assert np.array_equal(bits(f(v, r, it)), bits(g["output"]))
    assert np.array_equal(bits(oracle_lib.svt(v)), bits(g["svt"]))


def test_3d_oracle_known_answers(oracle_lib):
    c = np.full((5, 6, 7), 3.0)
    for r in (1, 2):  # test_filters3d.cpp:71-82: constants are fixed points
        assert np.array_equal(oracle_lib.osbf_3d(c, r, 2), c)
        assert np.array_equal(oracle_lib.box_filter_3d(c, r, 2), c)
    for r, it in ((0, 0), (1, -1)):
        with pytest.raises(oracle.CheckerError):
            oracle_lib.osbf_3d(c, r, it)


def test_3d_oracle_matches_compiled_reference(oracle_lib, reference_lib):
    rng = np.random.default_rng(64)
    for _ in range(3):
        shape = tuple(int(v) for v in rng.integers(1, 12, 3))
        r = int(rng.choice([1, 2, 4]))
        v = rng.random(shape) * 10
        assert np.array_equal(bits(oracle_lib.osbf_3d(v, r, 2)),
                              bits(reference_lib.osbf_3d(v, r, 2)))
        assert np.array_equal(bits(oracle_lib.box_filter_3d(v, r, 2)),
                              bits(reference_lib.box_filter_3d(v, r, 2)))


@pytest.mark.gpu
@pytest.mark.parametrize("path", filter3d_golden_cases(), ids=os.path.basename)
def test_3d_gpu_matches_reference_golden(ctx, path):
    import torch

    g = load_golden(path)
    v, r, it = g["input"], int(g["radius"]), int(g["iterations"])
    osbf3 = bool(g["osbf3"])
    dv = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).cuda()
    got = (ctx.osbf_3d(dv, r, it) if osbf3 else ctx.box_filter_3d(dv, r, it)).cpu().numpy()
    assert np.array_equal(bits(got), bits(g["output"]))
    assert np.array_equal(bits(ctx.filter3d_host(v, r, it, osbf3=osbf3)), bits(g["output"]))
    svt = ctx.svt_host(v)
    assert np.array_equal(bits(svt.reshape(-1)), bits(np.asarray(g["svt"]).reshape(-1)))


@pytest.mark.gpu
def test_3d_gpu_random_and_errors(ctx, oracle_lib):
    import torch

    import paper_2108_05021_b200 as ob

    rng = np.random.default_rng(65)
    for shape, r in (((20, 33, 41), 2), ((3, 70, 9), 5), ((1, 1, 1), 1)):
        v = rng.random(shape) * 255
        got = ctx.osbf_3d(torch.from_numpy(v).cuda(), r, 2).cpu().numpy()
        assert np.array_equal(bits(got), bits(oracle_lib.osbf_3d(v, r, 2)))
        got = ctx.box_filter_3d(torch.from_numpy(v).cuda(), r, 2).cpu().numpy()
        assert np.array_equal(bits(got), bits(oracle_lib.box_filter_3d(v, r, 2)))
        assert np.array_equal(bits(ctx.svt_host(v)), bits(oracle_lib.svt(v)))
    with pytest.raises(ob.InvalidArgument):
        ob.osbf_3d(np.ones((2, 2, 2)), 0, 0)
    with pytest.raises(ob.InvalidArgument):
        ob.box_filter_3d(np.ones((2, 2, 2)), 1, -1)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(300, 200, 5), (260, 128, 3), (257, 129, 9), (140, 133, 4),
                                   (129, 1, 7), (1, 300, 2), (2, 2, 37), (513, 7, 1)],
                         ids=lambda s: "x".join(map(str, s)))
def test_svt_wavefront_regimes_bit_exact(ctx, oracle_lib, shape):
    """osbf_3d.cu svt_yz: plane slots restart every Hp steps (H below, at and
    just above the 128 slots; several wraps over z) — bit-identical tables."""
    rng = np.random.default_rng(sum(shape))
    v = rng.random(shape) * 255
    assert np.array_equal(bits(ctx.svt_host(v)), bits(oracle_lib.svt(v)))
