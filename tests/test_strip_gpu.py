"""Fast mode through the persistent strip walker (osbf_strip.cuh), the
kernel every TMA-describable fast pass runs: parity with the reference
(oracle) at every compiled radius on shapes that take this path, the uint8
first pass bit-exact, and results independent of how the work is split
(bands, row bands of a multi-GPU split, batch chunks).
"""
import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def strip_kernel():
    """Force the strip walker for every fast pass of these tests."""
    import paper_2108_05021_b200 as ob

    ob.Context.set_fast_kernel("strip")
    yield
    ob.Context.set_fast_kernel(None)

FLOAT_TOL = 1e-5  # north_star: max-abs <= 1e-5 of the value range


def dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# widths multiple of 16 (the 4-D TMA view's group), heights around the
# radius, the chunk, a band; batches
SHAPES = [(1, 1, 16), (1, 5, 16), (2, 33, 48), (1, 300, 256), (3, 67, 272), (1, 1100, 528)]


@pytest.mark.parametrize("r", range(1, 17))
def test_strip_every_radius(ctx, oracle_lib, r):
    rng = np.random.default_rng(4000 + r)
    for shape in SHAPES:
        p = rng.random(shape) * 255.0
        got = ctx.iterate(dev(p), r, 3, mode="fast").cpu().numpy()
        assert ctx.last_kernel == "fast_strip", (shape, ctx.last_kernel)
        want = np.stack([oracle_lib.osbf(c, r, 3, threads=8) for c in p])
        err = float(np.abs(got - want).max())
        assert err <= FLOAT_TOL * 255.0, (shape, err)
    # uint8 first pass: integer sums, IEEE divisions -> bit-exact
    u8 = rng.integers(0, 256, (2, 140, 320), dtype=np.uint8)
    got = ctx.iterate(dev(u8), r, 1, mode="fast").cpu().numpy()
    assert ctx.last_kernel == "fast_strip"
    want = np.stack([oracle_lib.osbf(c.astype(np.float64), r, 1) for c in u8])
    assert np.array_equal(bits(got), bits(want))
    # float32 input read in its own dtype on the first pass
    f32 = (rng.random((1, 90, 160)) * 4 - 2).astype(np.float32)
    got = ctx.iterate(dev(f32), r, 2, mode="fast").cpu().numpy()
    want = oracle_lib.osbf(f32[0].astype(np.float64), r, 2)
    assert float(np.abs(got[0] - want).max()) <= FLOAT_TOL * 4.0


@pytest.mark.parametrize("r", [1, 2, 3, 4, 6, 8, 11, 16])
def test_strip_batch_chunks_bit_identical(ctx, r):
    """A batch filtered at once equals its planes filtered one by one."""
    import torch

    rng = np.random.default_rng(50 + r)
    p = rng.random((5, 200, 512))
    whole = ctx.iterate(dev(p), r, 2, mode="fast").cpu().numpy()
    for i in range(5):
        one = ctx.iterate(dev(p[i]), r, 2, mode="fast").cpu().numpy()
        assert np.array_equal(bits(one), bits(whole[i]))
    torch.cuda.synchronize()


@pytest.mark.parametrize("r", [1, 2, 4, 8, 12, 16])
def test_strip_row_bands(ctx, r):
    """Row-band passes (the multi-GPU split: each band reads its halo rows,
    windows clip at the global border) equal the whole-image pass: bit for
    bit for band starts aligned to the chunk rows (radii with register
    rings), within fp64 rounding otherwise."""
    import torch

    rng = np.random.default_rng(77 + r)
    H, W = 1000, 512
    p = dev(rng.random((H, W)) * 100.0)
    whole = ctx.iterate(p, r, 1, mode="fast")
    for cuts in ([0, 320, 640, H], [0, 333, 700, H]):
        out = torch.empty((H, W), dtype=torch.float64, device="cuda")
        for a, b in zip(cuts[:-1], cuts[1:]):
            i0, i1 = max(0, a - r), min(H, b + r)
            ctx.step_band(p[i0:i1], i0, out[a:b], a, b - a, H, r)
            assert ctx.last_kernel == "fast_strip"
        diff = float((out - whole).abs().max())
        aligned = all(c % 16 == 0 for c in cuts[1:-1])
        if aligned and r <= 8:
            assert diff == 0.0, (cuts, diff)
        else:
            assert diff <= 1e-9 * 100.0, (cuts, diff)


def test_strip_fused_push_matches_whole(ctx):
    """The halo push fused into the pass (row bands writing their edge rows
    into the neighbours' halo buffers): emulate three ranks on one device,
    passes issued one after another (no kernel waits on another)."""
    import torch

    r, H, W, iters = 4, 768, 512, 5
    rng = np.random.default_rng(9)
    x = dev(rng.random((H, W)))
    want = ctx.iterate(x, r, iters, mode="fast")
    cuts = [0, 256, 512, H]
    bufs = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        top, bot = (r if a > 0 else 0), (r if b < H else 0)
        buf = torch.zeros((b - a + top + bot, W), dtype=torch.float64, device="cuda")
        buf.copy_(x[a - top:b + bot])
        bufs.append([buf, top, bot, a, b])
    nxt = [torch.empty_like(bb[0]) for bb in bufs]
    for _ in range(iters):
        for i, (buf, top, bot, a, b) in enumerate(bufs):
            dst = nxt[i]
            up = nxt[i - 1][-r:] if i > 0 else None  # upper neighbour's bottom halo
            dn = nxt[i + 1][:r] if i + 1 < len(bufs) else None
            ctx.step_band(buf, a - top, dst[top:top + b - a], a, b - a, H, r,
                          push_up=up, push_down=dn, push_rows=r if (up is not None or dn is not None) else 0)
        for i in range(len(bufs)):
            bufs[i][0], nxt[i] = nxt[i], bufs[i][0]
    got = torch.cat([bb[0][bb[1]:bb[1] + bb[4] - bb[3]] for bb in bufs])
    assert torch.equal(got.view(torch.int64), want.view(torch.int64))
