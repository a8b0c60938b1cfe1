"""Every exact-pass kernel family (osbf_gpu_set_exact_kernel): the fused
strip walk, and the whole-table path with the generic walk (default), the
templated walk or the per-thread stencil.  All must be bit-identical to the
reference (oracle) -- and therefore to each other -- on the same inputs."""
import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu

FAMILIES = {"strip": "exact_strip", "gwalk": "exact_gwalk", "twalk": "exact_twalk",
            "stencil": "exact_select"}


def dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(params=sorted(FAMILIES))
def family(request):
    import paper_2108_05021_b200 as ob

    ob.Context.set_exact_kernel(request.param)
    yield request.param
    ob.Context.set_exact_kernel(None)


@pytest.mark.parametrize("shape,r", [((1, 300, 260), 1), ((3, 130, 272), 2), ((2, 97, 400), 5),
                                     ((1, 700, 144), 8), ((40, 64, 64), 3), ((1, 260, 300), 16)])
def test_exact_family_matches_oracle(ctx, oracle_lib, family, shape, r):
    rng = np.random.default_rng(sum(shape) * 7 + r)
    p = rng.random(shape) * 255.0
    got = ctx.iterate(dev(p), r, 3, mode="exact").cpu().numpy()
    assert FAMILIES[family] in ctx.last_kernel
    want = np.stack([oracle_lib.osbf(c, r, 3) for c in p])
    assert np.array_equal(bits(got), bits(want))


def test_exact_family_uint8_first_pass_and_ties(ctx, oracle_lib, family):
    p = np.zeros((200, 256), dtype=np.uint8)
    p[:, 100:] = 180
    p[50:150, 60:200] = 40
    p[::9, ::4] = 255
    got = ctx.iterate(dev(p), 3, 5, mode="exact").cpu().numpy()
    assert np.array_equal(bits(got), bits(oracle_lib.osbf(p.astype(np.float64), 3, 5)))


def test_unknown_exact_family_is_rejected():
    import paper_2108_05021_b200 as ob

    with pytest.raises(ob.InvalidArgument):
        ob.Context.set_exact_kernel("nope")


def test_non_finite_image_does_not_slow_later_ones(ctx, oracle_lib):
    """The table's 'unsafe' word is per pass: after a NaN image, a finite image
    is again served by the unguarded path (same bits either way; checked
    through the result, and through the flag-free default kernels running)."""
    rng = np.random.default_rng(3)
    bad = rng.random((128, 256)) * 10.0
    bad[7, 9] = np.nan
    got = ctx.iterate(dev(bad), 2, 2, mode="exact").cpu().numpy()
    assert np.array_equal(bits(got), bits(oracle_lib.osbf(bad, 2, 2)))
    good = rng.random((128, 256)) * 10.0
    got = ctx.iterate(dev(good), 2, 2, mode="exact").cpu().numpy()
    assert np.array_equal(bits(got), bits(oracle_lib.osbf(good, 2, 2)))


@pytest.mark.parametrize("dtype", [np.uint8, np.float32, np.float64])
@pytest.mark.parametrize("shape", [(1, 300, 260), (2, 97, 1024), (3, 33, 31), (1, 70, 32),
                                   (1, 64, 33), (40, 40, 50)])
def test_table_builders_agree(ctx, oracle_lib, dtype, shape):
    """The summed-area table (osbf_gpu_sat: strip builder = row carries +
    exact_table_strip; widths around the 32-column strip edges, partial tiles,
    several planes) is the reference's table bit for bit, for every input
    dtype -- the strip builder's register-staged path for uint8 / float32."""
    rng = np.random.default_rng(sum(shape) + np.dtype(dtype).itemsize)
    if dtype == np.uint8:
        p = rng.integers(0, 256, shape, dtype=np.uint8)
    else:
        p = (rng.random(shape) * 255.0 - 40.0).astype(dtype)
    for plane in p:
        got = ctx.sat(dev(plane)).cpu().numpy()
        want = oracle_lib.sat(plane.astype(np.float64))
        assert np.array_equal(bits(got), bits(want))
    # and through a pass (own even-pitch table + flag word)
    got = ctx.iterate(dev(p), 2, 2, mode="exact").cpu().numpy()
    want = np.stack([oracle_lib.osbf(c.astype(np.float64), 2, 2) for c in p])
    assert np.array_equal(bits(got), bits(want))
