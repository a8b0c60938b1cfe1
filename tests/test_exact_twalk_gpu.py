"""Exact mode, whole-table path with the TMA-staged stencil walk
(osbf_exact_twalk.cuh): bit-identical to the reference (oracle) on every
radius the walk is compiled for, every input dtype, clipped borders, row
blocks, several planes, and non-finite samples (guarded fallback).

The templated walk is a selectable family (the default stencil is the
generic-radius walk, osbf_exact_gwalk.cuh), forced here; widths whose rows
are not 16-byte multiples fall back to the per-thread stencil, so both are
covered."""
import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def twalk_family():
    import paper_2108_05021_b200 as ob

    ob.Context.set_exact_kernel("twalk")
    yield
    ob.Context.set_exact_kernel(None)


def dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def want(oracle_lib, p, r, it):
    planes = p.reshape((-1,) + p.shape[-2:])
    return np.stack([oracle_lib.osbf(c, r, it) for c in planes]).reshape(p.shape)


@pytest.mark.parametrize("r", list(range(1, 17)))
def test_twalk_every_radius_f64(ctx, oracle_lib, r):
    rng = np.random.default_rng(500 + r)
    p = rng.random((300, 260)) * 255.0  # 3 strips (last partial), 2 row blocks
    got = ctx.iterate(dev(p), r, 3, mode="exact").cpu().numpy()
    assert "twalk" in ctx.last_kernel
    assert np.array_equal(bits(got), bits(want(oracle_lib, p, r, 3)))


@pytest.mark.parametrize("dtype,w", [(np.uint8, 272), (np.float32, 132), (np.float64, 130)])
@pytest.mark.parametrize("r", [2, 5, 16])
def test_twalk_input_dtypes(ctx, oracle_lib, dtype, w, r):
    rng = np.random.default_rng(7 * r + w)
    if dtype == np.uint8:
        p = rng.integers(0, 256, (211, w), dtype=np.uint8)
    else:
        p = (rng.random((211, w)) * 255.0).astype(dtype)
    got = ctx.iterate(dev(p), r, 2, mode="exact").cpu().numpy()
    assert np.array_equal(bits(got), bits(want(oracle_lib, p.astype(np.float64), r, 2)))


@pytest.mark.parametrize("shape", [(3, 97, 200), (2, 600, 128), (1, 5, 40), (1, 40, 6)])
def test_twalk_planes_and_small_shapes(ctx, oracle_lib, shape):
    rng = np.random.default_rng(sum(shape))
    p = rng.random(shape) * 100.0 - 20.0  # mixed signs
    for r in (1, 3, 8):
        got = ctx.iterate(dev(p), r, 2, mode="exact").cpu().numpy()
        assert np.array_equal(bits(got), bits(want(oracle_lib, p, r, 2))), r


def test_twalk_uint8_ties(ctx, oracle_lib):
    """Flat and two-level uint8 regions: exact ties between windows decided
    by the table's rounding noise after the first pass."""
    p = np.zeros((256, 256), dtype=np.uint8)
    p[:, 128:] = 200
    p[64:192, 64:192] = 50
    p[::7, ::5] = 255
    got = ctx.iterate(dev(p), 4, 6, mode="exact").cpu().numpy()
    assert np.array_equal(bits(got), bits(want(oracle_lib, p.astype(np.float64), 4, 6)))


def test_twalk_non_finite_and_huge(ctx, oracle_lib):
    """NaN / inf samples and values beyond the unguarded division's range:
    the chain kernels raise the table flag and the walk takes the guarded
    per-window rule for every pixel."""
    rng = np.random.default_rng(9)
    p = rng.random((140, 256)) * 30.0
    p[5, 7] = np.nan
    p[100, 200] = np.inf
    got = ctx.iterate(dev(p), 2, 2, mode="exact").cpu().numpy()
    assert np.array_equal(bits(got), bits(want(oracle_lib, p, 2, 2)))
    q = rng.random((64, 128)) * 1e300
    got = ctx.iterate(dev(q), 3, 1, mode="exact").cpu().numpy()
    assert np.array_equal(bits(got), bits(want(oracle_lib, q, 3, 1)))
