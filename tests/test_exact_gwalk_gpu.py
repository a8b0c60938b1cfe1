"""Exact mode, whole-table path, radii above the templated walk (r = 17..62):
the generic-radius stencil walk (osbf_exact_gwalk.cuh) streams the four table
rows a pixel reads through three TMA row streams.  Bit-identical to the
reference (oracle) for every radius class, input dtype, clipped borders
(windows wider than the image included), several planes and non-finite
samples; widths TMA cannot describe fall back to the per-thread stencil."""
import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu


def dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def want(oracle_lib, p, r, it):
    planes = p.reshape((-1,) + p.shape[-2:])
    return np.stack([oracle_lib.osbf(c, r, it) for c in planes]).reshape(p.shape)


@pytest.mark.parametrize("r", [17, 18, 24, 31, 32, 47, 61, 62])
def test_gwalk_radii_f64(ctx, oracle_lib, r):
    rng = np.random.default_rng(900 + r)
    p = rng.random((300, 260)) * 255.0  # 3 strips (last partial), several row blocks
    got = ctx.iterate(dev(p), r, 2, mode="exact").cpu().numpy()
    assert "gwalk" in ctx.last_kernel
    assert np.array_equal(bits(got), bits(want(oracle_lib, p, r, 2)))


def test_gwalk_beyond_its_radius_runs_stencil(ctx, oracle_lib):
    rng = np.random.default_rng(63)
    p = rng.random((150, 136)) * 255.0
    got = ctx.iterate(dev(p), 63, 1, mode="exact").cpu().numpy()
    assert "exact_select" in ctx.last_kernel
    assert np.array_equal(bits(got), bits(want(oracle_lib, p, 63, 1)))


@pytest.mark.parametrize("dtype,w", [(np.uint8, 272), (np.float32, 132), (np.float64, 130)])
@pytest.mark.parametrize("r", [20, 33])
def test_gwalk_input_dtypes(ctx, oracle_lib, dtype, w, r):
    rng = np.random.default_rng(7 * r + w)
    if dtype == np.uint8:
        p = rng.integers(0, 256, (211, w), dtype=np.uint8)
    else:
        p = (rng.random((211, w)) * 255.0).astype(dtype)
    got = ctx.iterate(dev(p), r, 2, mode="exact").cpu().numpy()
    assert "gwalk" in ctx.last_kernel
    assert np.array_equal(bits(got), bits(want(oracle_lib, p.astype(np.float64), r, 2)))


@pytest.mark.parametrize("shape", [(3, 97, 200), (2, 600, 128), (1, 5, 40), (1, 40, 6),
                                   (70, 64, 64)])
def test_gwalk_planes_and_windows_wider_than_the_image(ctx, oracle_lib, shape):
    rng = np.random.default_rng(sum(shape))
    p = rng.random(shape) * 100.0 - 20.0  # mixed signs
    for r in (17, 40):
        got = ctx.iterate(dev(p), r, 2, mode="exact").cpu().numpy()
        assert np.array_equal(bits(got), bits(want(oracle_lib, p, r, 2))), r


def test_gwalk_unaligned_width_falls_back(ctx, oracle_lib):
    """uint8 rows that are not 16-byte multiples cannot be TMA-staged."""
    rng = np.random.default_rng(5)
    p = rng.integers(0, 256, (90, 150), dtype=np.uint8)
    got = ctx.iterate(dev(p), 20, 1, mode="exact").cpu().numpy()
    assert "exact_select" in ctx.last_kernel
    assert np.array_equal(bits(got), bits(want(oracle_lib, p.astype(np.float64), 20, 1)))


def test_gwalk_uint8_ties(ctx, oracle_lib):
    p = np.zeros((256, 256), dtype=np.uint8)
    p[:, 128:] = 200
    p[64:192, 64:192] = 50
    p[::7, ::5] = 255
    got = ctx.iterate(dev(p), 20, 4, mode="exact").cpu().numpy()
    assert np.array_equal(bits(got), bits(want(oracle_lib, p.astype(np.float64), 20, 4)))


def test_gwalk_non_finite_and_huge(ctx, oracle_lib):
    """NaN / inf samples and values beyond the unguarded division's range
    raise the table flag: every pixel then takes the guarded per-window rule.
    (Runs last in this module: the flag is sticky for the process.)"""
    rng = np.random.default_rng(9)
    p = rng.random((140, 256)) * 30.0
    p[5, 7] = np.nan
    p[100, 200] = np.inf
    got = ctx.iterate(dev(p), 18, 2, mode="exact").cpu().numpy()
    assert np.array_equal(bits(got), bits(want(oracle_lib, p, 18, 2)))
    q = rng.random((64, 128)) * 1e300
    got = ctx.iterate(dev(q), 19, 1, mode="exact").cpu().numpy()
    assert np.array_equal(bits(got), bits(want(oracle_lib, q, 19, 1)))
