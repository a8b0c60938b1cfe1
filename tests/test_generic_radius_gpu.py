"""Fast mode above the templated radii (r > 16): the generic vertical-first
walk (osbf_fast_vwalk.cu) against the oracle on ragged shapes, uint8 first
pass bit-exact, row bands, and the exact fallback beyond its largest radius
(the reference accepts any r >= 1, filters2d.hpp:61-63)."""
import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu

FLOAT_TOL = 1e-5


def test_generic_max_radius_host_query():
    import paper_2108_05021_b200 as ob

    assert ob.Context.fast_max_radius() >= 64


@pytest.fixture
def vwalk():
    """Small test planes would not fill one wave of CTAs, where whole-plane
    calls prefer the exact path: force the generic walk."""
    import paper_2108_05021_b200 as ob

    ob.Context.set_fast_kernel("vwalk")
    yield
    ob.Context.set_fast_kernel(None)


@pytest.mark.parametrize("r", [17, 20, 24, 32, 47, 56])
def test_generic_radius_matches_oracle(ctx, oracle_lib, vwalk, r):
    import torch
    rng = np.random.default_rng(1700 + r)
    for shape in [(1, 3, 2), (1, r, 2 * r + 1), (2, 37, 300), (1, 700, 129), (1, 530, 611)]:
        p = rng.random(shape) * 255.0
        got = ctx.iterate(torch.from_numpy(p).cuda(), r, 3, mode="fast").cpu().numpy()
        assert ctx.last_kernel == "fast_vwalk_step", shape  # odd widths: plain loads
        want = np.stack([oracle_lib.osbf(c, r, 3) for c in p])
        assert float(np.abs(got - want).max()) <= FLOAT_TOL * 255.0, shape
    u8 = rng.integers(0, 256, (2, 300, 290), dtype=np.uint8)
    got = ctx.iterate(torch.from_numpy(u8).cuda(), r, 1, mode="fast").cpu().numpy()
    want = np.stack([oracle_lib.osbf(c.astype(np.float64), r, 1) for c in u8])
    assert np.array_equal(bits(got), bits(want))
    f32 = (rng.random((1, 200, 333)) * 8 - 4).astype(np.float32)
    got = ctx.iterate(torch.from_numpy(f32).cuda(), r, 2, mode="fast").cpu().numpy()
    want = oracle_lib.osbf(f32[0].astype(np.float64), r, 2)
    assert float(np.abs(got[0] - want).max()) <= FLOAT_TOL * 8.0


def test_generic_radius_tall_image_blocks(ctx, oracle_lib, vwalk):
    """Several 512-row blocks per strip and several strips (block seams)."""
    import torch

    r = 21
    p = np.random.default_rng(5).random((1300, 300)) * 100.0
    got = ctx.iterate(torch.from_numpy(p).cuda(), r, 2, mode="fast").cpu().numpy()
    want = oracle_lib.osbf(p, r, 2)
    assert float(np.abs(got - want).max()) <= FLOAT_TOL * 100.0


@pytest.mark.parametrize("r", [20, 40])
def test_generic_radius_row_bands(ctx, vwalk, r):
    """Row bands on the 512-row block grid are bit-identical to the whole
    image; other cuts agree to fp64 rounding."""
    import torch

    from paper_2108_05021_b200.dist import BandLayout

    h, w, iters = 1536 + 77, 260, 2
    x = torch.from_numpy(np.random.default_rng(60 + r).random((h, w))).cuda()
    want = ctx.iterate(x, r, iters, mode="fast")
    for world, exact in ((3, True), (4, False)):
        cur = x.clone()
        for _ in range(iters):
            nxt = torch.empty_like(cur)
            for rank in range(world):
                lay = BandLayout.make(h, w, r, world, rank)
                src = cur[lay.buf_row0:lay.buf_row0 + lay.buf_rows].contiguous()
                ctx.step_band(src, lay.buf_row0, nxt[lay.row0:lay.row1], lay.row0, lay.rows, h, r)
            cur = nxt
        if exact:
            assert torch.equal(cur.view(torch.int64), want.view(torch.int64))
        else:
            assert float((cur - want).abs().max()) <= 1e-9


@pytest.mark.parametrize("r", [57, 100])
def test_generic_radius_row_bands_large(ctx, oracle_lib, r):
    """Bands keep the generic walk up to fast_max_radius() (the exact path
    cannot be banded): 3 bands of a 2-pass run within the float tolerance."""
    import torch

    from paper_2108_05021_b200.dist import BandLayout

    h, w, iters, world = 700, 2 * r + 40, 2, 3
    p = np.random.default_rng(r).random((h, w)) * 10.0
    cur = torch.from_numpy(p).cuda()
    for _ in range(iters):
        nxt = torch.empty_like(cur)
        for rank in range(world):
            lay = BandLayout.make(h, w, r, world, rank)
            src = cur[lay.buf_row0:lay.buf_row0 + lay.buf_rows].contiguous()
            ctx.step_band(src, lay.buf_row0, nxt[lay.row0:lay.row1], lay.row0, lay.rows, h, r)
        cur = nxt
    assert ctx.last_kernel == "fast_vwalk_step"
    want = oracle_lib.osbf(p, r, iters)
    assert float(np.abs(cur.cpu().numpy() - want).max()) <= FLOAT_TOL * 10.0


def test_beyond_generic_radius_runs_exact(ctx, oracle_lib):
    import torch

    r = 57
    p = np.random.default_rng(3).random((40, 2 * r + 5)) * 10.0
    got = ctx.iterate(torch.from_numpy(p).cuda(), r, 2, mode="fast").cpu().numpy()
    assert "exact" in ctx.last_kernel
    assert np.array_equal(bits(got), bits(oracle_lib.osbf(p, r, 2)))


def test_whole_planes_above_16_run_the_exact_table_path(ctx, oracle_lib):
    """Whole planes at r > 16 run the exact kernels in fast mode too: they are
    bit-identical to the reference and, since the strip table builder and the
    generic stencil walk, faster than the generic fast walk at every such
    radius (the walk serves row bands and can be forced)."""
    import torch

    for shape in ((300, 260), (2048, 2048)):
        p = np.random.default_rng(8).random(shape) * 10.0
        got = ctx.iterate(torch.from_numpy(p).cuda(), 20, 2, mode="fast").cpu().numpy()
        assert "exact_gwalk" in ctx.last_kernel
        assert np.array_equal(bits(got), bits(oracle_lib.osbf(p, 20, 2, threads=8)))


def test_large_plane_generic_walk_forced(ctx, oracle_lib, vwalk):
    import torch

    p = np.random.default_rng(9).random((8192, 8192)) * 10.0  # 64 strips x 16 blocks
    got = ctx.iterate(torch.from_numpy(p).cuda(), 20, 1, mode="fast").cpu().numpy()
    assert ctx.last_kernel == "fast_vwalk_step"
    want = oracle_lib.osbf(p, 20, 1, threads=8)
    assert float(np.abs(got - want).max()) <= FLOAT_TOL * 10.0
