"""GPU parity on the BASELINE.json configurations the benchmark numbers are
quoted on, at their full sizes, against the CPU oracle (the C restatement,
itself pinned bit-for-bit to the unmodified reference, tests/test_oracle.py).

  C3  4096^2 uint8, 10 iterations, r in {1,2,4,8,16}: exact mode bit-exact
      (the row-band exact path of a single large plane); fast mode's first
      pass bit-exact (integer sums)
  C4  1024^2 float32 planes (2 rectangle + 2 polygon mosaics), r=2, 20
      iterations: exact bit-exact, fast within 1e-5 of the value range
  C5  32768^2 float32, r=4: 2 iterations over the whole image, exact mode
      bit-exact; fast mode within tolerance except near ties that the
      reference's own whole-image table rounding decides (classified pixel by
      pixel, see near_tie_flips); 50 fast iterations over a 32768 x 4096
      band (the weak-scaling per-GPU image), and the same band split into two
      row bands with the halo exchange bit-identical to the whole
"""
import os

import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu

FLOAT_TOL = 1e-5
THREADS = os.cpu_count() or 1


def dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def vrange(a):
    return float(np.max(a) - np.min(a))


@pytest.mark.parametrize("r", [1, 2, 4, 8, 16])
def test_c3_full_exact_bit_exact(ctx, oracle_lib, r):
    from paper_2108_05021_b200 import synth

    x = synth.make_input("C3")[0]  # 4096 x 4096 uint8
    got = ctx.iterate(dev(x), r, 10, mode="exact").cpu().numpy()
    want = oracle_lib.osbf(x.astype(np.float64), r, 10, threads=THREADS)
    assert np.array_equal(bits(got), bits(want))
    one = ctx.iterate(dev(x), r, 1, mode="fast").cpu().numpy()
    assert np.array_equal(bits(one), bits(oracle_lib.osbf(x.astype(np.float64), r, 1,
                                                          threads=THREADS)))


def test_c4_planes_full_20_iterations(ctx, oracle_lib):
    from paper_2108_05021_b200 import synth

    planes = np.stack([synth.c4_plane(i) for i in range(4)])  # rect, poly, rect, poly
    want = np.stack([oracle_lib.osbf(p.astype(np.float64), 2, 20, threads=THREADS)
                     for p in planes])
    exact = ctx.iterate(dev(planes), 2, 20, mode="exact").cpu().numpy()
    assert np.array_equal(bits(exact), bits(want))
    fast = ctx.iterate(dev(planes), 2, 20, mode="fast").cpu().numpy()
    for i in range(4):
        err = float(np.abs(fast[i] - want[i]).max())
        assert err <= FLOAT_TOL * vrange(planes[i]), (i, err)


def _host_ram_gb():
    try:
        import psutil

        return psutil.virtual_memory().available / 2**30
    except Exception:  # noqa: BLE001
        return 0.0


@pytest.fixture(scope="module")
def c5_input():
    from paper_2108_05021_b200 import synth

    return synth.make_input("C5")[0]  # 32768 x 32768 float32, seeded


def near_tie_flips(oracle_lib, plane, got, want, r, tol):
    """Fast-mode disagreements with the reference on one pass, classified.

    The reference sums every window from ONE whole-image fp64 table; on a
    32768^2 image its entries reach ~5e8, so its window sums carry ~1e-7 of
    rounding noise, and where two windows' |a - u| are that close (opposite
    sides of u) that noise, not the data, decides the winner.  Every pixel
    where the fast pass (exactly summed local windows) differs from the
    reference beyond ``tol`` must be such a near tie: the fast output is
    another window's reference mean, and that window's |a - u| is within
    1e-6 of the reference's winner.  Returns the number of such pixels."""
    bad = np.argwhere(np.abs(got - want) > tol)
    if len(bad) == 0:
        return 0
    h, w = plane.shape
    cs = oracle_lib.sat(plane)
    for y, x in bad[:4000]:
        m = oracle_lib.subwindow_means(cs, w, h, int(x), int(y), r)
        d = np.abs(m - plane[y, x])
        k = int(np.argmin(np.abs(m - got[y, x])))
        assert abs(m[k] - got[y, x]) <= tol, (y, x, m, got[y, x])
        assert d[k] - d.min() <= 1e-6, (y, x, d)
    return len(bad)


@pytest.mark.skipif(_host_ram_gb() < 48, reason="the C5 oracle needs ~35 GB of host RAM")
def test_c5_full(ctx, oracle_lib, c5_input):
    """The whole 32768^2 image, r=4: exact mode bit-exact over 2 passes; fast
    mode's first pass within tolerance except near-tie flips decided by the
    reference's table rounding (see near_tie_flips), at most 1e-5 of the
    pixels; after 2 passes at most 1e-4 of the pixels beyond tolerance (a
    flip moves its neighbours' sums in the next pass)."""
    import torch

    x = dev(c5_input)
    fast1 = ctx.iterate(x, 4, 1, mode="fast").cpu().numpy()
    fast2 = ctx.iterate(x, 4, 2, mode="fast").cpu().numpy()
    exact = ctx.iterate(x, 4, 2, mode="exact").cpu().numpy()
    del x
    torch.cuda.empty_cache()
    plane = c5_input.astype(np.float64)
    want2 = oracle_lib.osbf(plane, 4, 2, threads=THREADS)
    assert np.array_equal(bits(exact), bits(want2))
    del exact
    tol = FLOAT_TOL * vrange(c5_input)
    want1 = oracle_lib.osbf(plane, 4, 1, threads=THREADS)
    flips = near_tie_flips(oracle_lib, plane, fast1, want1, 4, tol)
    assert flips <= 1e-5 * plane.size, flips
    beyond = int(np.count_nonzero(np.abs(fast2 - want2) > tol))
    print(f"\nC5 fast vs reference: pass 1 {flips} near-tie flips of {plane.size} px; "
          f"2 passes {beyond} px beyond {tol:.3g}")
    assert beyond <= 1e-4 * plane.size, beyond


def test_c5_band_50_iterations(ctx, oracle_lib, c5_input):
    """The weak-scaling per-GPU image (32768 wide x 4096 rows of C5), r=4,
    50 fast passes: within tolerance of the oracle; and as two row bands
    (each pass reads the neighbour's halo rows, windows clip at the global
    border) bit-identical to the whole."""
    import torch

    band = np.ascontiguousarray(c5_input[:4096])
    x = dev(band)
    whole = ctx.iterate(x, 4, 50, mode="fast")
    want = oracle_lib.osbf(band.astype(np.float64), 4, 50, threads=THREADS)
    tol = FLOAT_TOL * vrange(band)
    beyond = int(np.count_nonzero(np.abs(whole.cpu().numpy() - want) > tol))
    assert beyond <= 1e-4 * band.size, beyond  # near-tie flips, see test_c5_full
    one = ctx.iterate(x, 4, 1, mode="fast").cpu().numpy()
    plane = band.astype(np.float64)
    flips = near_tie_flips(oracle_lib, plane, one,
                           oracle_lib.osbf(plane, 4, 1, threads=THREADS), 4, tol)
    print(f"\nC5 band fast vs reference: pass 1 {flips} near-tie flips; "
          f"50 passes {beyond} of {band.size} px beyond {tol:.3g}")

    # two row bands [0, 2048) and [2048, 4096), r-row halo exchanged per pass
    r, H, W = 4, 4096, 32768
    cur = x.double()
    nxt = torch.empty_like(cur)
    for _ in range(50):
        for a, b in ((0, 2048), (2048, H)):
            i0, i1 = max(0, a - r), min(H, b + r)
            ctx.step_band(cur[i0:i1], i0, nxt[a:b], a, b - a, H, r)
        cur, nxt = nxt, cur
    assert torch.equal(cur.view(torch.int64), whole.view(torch.int64))
