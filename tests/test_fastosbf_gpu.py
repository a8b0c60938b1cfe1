"""Paper Algorithm 3 on the GPU (osbf_gpu_fast_osbf): bit-identical to the
reference's fast_osbf (filters2d.hpp:105-154) — golden outputs of the
unmodified reference, the oracle on random shapes / radii / dtypes, the
reference's error behaviour, and the OsbfFast branch of filter_multichannel
(filters2d.hpp:386)."""
import os

import numpy as np
import pytest

from conftest import bits, fastosbf_golden_cases, load_golden

pytestmark = pytest.mark.gpu


def dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("path", fastosbf_golden_cases(), ids=os.path.basename)
def test_fast_osbf_matches_reference_golden(ctx, path):
    import paper_2108_05021_b200 as ob

    g = load_golden(path)
    x, r, it = g["input"], int(g["radius"]), int(g["iterations"])
    if x.ndim == 3:  # filter_multichannel(OsbfFast)
        cfg = ob.FilterConfig(radius=r, iterations=it, variant=ob.FilterVariant.OsbfFast)
        host = np.stack(ob.filter_multichannel([c.astype(np.float64) for c in x], cfg))
        assert np.array_equal(bits(host), bits(g["output"]))
    got = ctx.fast_osbf(dev(x), r, it).cpu().numpy()
    assert np.array_equal(bits(got), bits(g["output"]))
    assert np.array_equal(bits(ctx.fast_osbf_host(x, r, it)), bits(g["output"]))


@pytest.mark.parametrize("seed", range(10))
def test_fast_osbf_random_shapes_bit_exact(ctx, oracle_lib, seed):
    rng = np.random.default_rng(700 + seed)
    h, w = int(rng.integers(1, 400)), int(rng.integers(1, 400))
    r = int(rng.choice([1, 2, 3, 4, 7, 16, 40, 70]))  # 70: the unfused field path
    p = rng.random((h, w)) * 255.0
    got = ctx.fast_osbf(dev(p), r, 3).cpu().numpy()
    assert np.array_equal(bits(got), bits(oracle_lib.fast_osbf(p, r, 3)))


def test_fast_osbf_dtypes_and_batch(ctx, oracle_lib):
    """uint8 / float32 inputs are promoted exactly; batch planes are independent."""
    from paper_2108_05021_b200 import synth

    rng = np.random.default_rng(5)
    u8 = synth.u8_mosaic(160, 120, rng, block=(4, 40))
    assert np.array_equal(bits(ctx.fast_osbf(dev(u8), 4, 5).cpu().numpy()),
                          bits(oracle_lib.fast_osbf(u8.astype(np.float64), 4, 5)))
    f32 = synth.make_input("C2", shrink=8)  # 3 channels, float32
    got = ctx.fast_osbf(dev(f32), 3, 4).cpu().numpy()
    for c in range(3):
        assert np.array_equal(bits(got[c]), bits(oracle_lib.fast_osbf(f32[c].astype(np.float64), 3, 4)))


def test_fast_osbf_errors(ctx):
    import paper_2108_05021_b200 as ob

    p = np.ones((8, 8))
    for r, it in ((0, 0), (0, 2), (2, -1)):
        with pytest.raises(ob.InvalidArgument):
            ob.fast_osbf(p, r, it)
    assert np.array_equal(ob.fast_osbf(p, 3, 0), p)


def test_fast_osbf_large_and_in_place(ctx, oracle_lib):
    import torch

    rng = np.random.default_rng(9)
    p = rng.random((1100, 1300))
    x = dev(p)
    want = oracle_lib.fast_osbf(p, 5, 2)
    assert np.array_equal(bits(ctx.fast_osbf(x, 5, 2).cpu().numpy()), bits(want))
    ctx.fast_osbf(x, 5, 2, out=x)  # in place
    assert np.array_equal(bits(x.cpu().numpy()), bits(want))
    assert x.dtype == torch.float64


def test_fast_osbf_tracks_exact_osbf(ctx):
    """acceptance.cpp:106-134 (criterion 4): RMSE(exact, fast) <= 5 on the
    0..255 scale for r in 2..10 at 1, 10, 50 iterations (a seeded mosaic +
    noise stands in for the reference's phantom image)."""
    import torch

    from paper_2108_05021_b200 import synth

    p = torch.from_numpy(synth.make_input("C1", shrink=2)[0].astype(np.float64) * 255.0).cuda()
    worst = 0.0
    for r in range(2, 11):
        e, f = p.clone(), p.clone()
        done = 0
        for checkpoint in (1, 10, 50):
            n = checkpoint - done
            e = ctx.iterate(e, r, n, mode="exact")
            f = ctx.fast_osbf(f, r, n)
            done = checkpoint
            worst = max(worst, float(torch.sqrt(torch.mean((e - f) ** 2))))
    assert worst <= 5.0, worst
