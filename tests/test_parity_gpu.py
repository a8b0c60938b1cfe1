"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and
the reference's golden outputs.

Bars (BASELINE.json north_star):
  * exact mode: bit-identical output and selection to the reference on every
    input, every iteration;
  * fast mode: bit-identical whenever window sums are exact (integer inputs,
    first pass); otherwise max-abs <= FLOAT_TOL * value range.
"""
import os

import numpy as np
import pytest

from conftest import bits, golden_cases, load_golden

pytestmark = pytest.mark.gpu

FLOAT_TOL = 1e-5  # north_star: max-abs error <= 1e-5 of the value range (float32 configs)


def torch_dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def vrange(a):
    a = np.asarray(a, dtype=np.float64)
    return max(float(a.max() - a.min()), 1e-300)


@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: os.path.basename(p)[:-4])
def test_exact_matches_reference_golden(ctx, path):
    g = load_golden(path)
    inp, r, it = g["input"], int(g["radius"]), int(g["iterations"])
    want = g["output"]
    got = ctx.iterate(torch_dev(inp), r, it, mode="exact").cpu().numpy()
    assert np.array_equal(bits(got), bits(want))
    # host-buffer entry point (what the drop-in C++ API calls)
    got_h = ctx.osbf_host(inp, r, it, mode="exact")
    assert np.array_equal(bits(got_h), bits(want))
    if it > 0:
        first = inp if inp.ndim == 2 else inp[0]
        means, sel = ctx.subwindow_means(torch_dev(first), r, mode="exact")
        assert np.array_equal(sel.cpu().numpy(), g["step1_sel"])
        if "step1_means" in g:
            assert np.array_equal(bits(means.cpu().numpy()), bits(g["step1_means"]))


@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: os.path.basename(p)[:-4])
def test_fast_matches_reference_golden(ctx, path):
    g = load_golden(path)
    inp, r, it = g["input"], int(g["radius"]), int(g["iterations"])
    got = ctx.iterate(torch_dev(inp), r, it, mode="fast").cpu().numpy()
    want = g["output"]
    if it == 0:
        assert np.array_equal(bits(got), bits(want))
        return
    if inp.dtype == np.uint8 or np.all(inp == np.round(inp)):
        # integer window sums are exact in any order: the first pass is bit-exact
        first = inp if inp.ndim == 2 else inp[0]
        one = ctx.iterate(torch_dev(first), r, 1, mode="fast").cpu().numpy()
        import oracle

        assert np.array_equal(bits(one), bits(oracle.Oracle().osbf(first, r, 1)))
    if inp.dtype != np.uint8:
        err = np.abs(got - want).max()
        assert err <= FLOAT_TOL * vrange(inp), f"max abs err {err}"


@pytest.mark.parametrize("seed", range(6))
def test_exact_random_shapes_bit_exact(ctx, oracle_lib, seed):
    rng = np.random.default_rng(100 + seed)
    h, w = int(rng.integers(1, 300)), int(rng.integers(1, 300))
    r = int(rng.choice([1, 2, 3, 4, 7, 16]))
    p = rng.random((h, w)) * 255.0
    got = ctx.iterate(torch_dev(p), r, 3, mode="exact").cpu().numpy()
    assert np.array_equal(bits(got), bits(oracle_lib.osbf(p, r, 3)))


@pytest.mark.parametrize("shape,r,scale", [
    ((1, 700, 333), 1, 255.0), ((1, 1000, 97), 2, 1.0), ((1, 2049, 40), 16, 1e6),
    ((3, 600, 200), 3, 255.0), ((1, 1537, 65), 8, 1e-300), ((2, 520, 31), 4, 1e300)])
def test_exact_row_bands_bit_exact(ctx, oracle_lib, shape, r, scale):
    """Tall planes with few 32-column strips run the exact strip kernel in
    row bands that start from stored table rows; must stay bit-exact,
    including values whose window divisions take the guarded path."""
    import paper_2108_05021_b200 as ob

    rng = np.random.default_rng(sum(shape) + r)
    p = rng.random(shape) * scale
    want = np.stack([oracle_lib.osbf(c, r, 2, threads=8) for c in p])
    ob.Context.set_exact_kernel("strip")  # (the default is the whole-table path)
    try:
        got = ctx.iterate(torch_dev(p), r, 2, mode="exact").cpu().numpy()
        assert "exact_strip" in ctx.last_kernel
    finally:
        ob.Context.set_exact_kernel(None)
    assert np.array_equal(bits(got), bits(want))
    got = ctx.iterate(torch_dev(p), r, 2, mode="exact").cpu().numpy()
    assert np.array_equal(bits(got), bits(want))


@pytest.mark.parametrize("r", range(1, 17))
def test_fast_every_radius_random_shapes(ctx, oracle_lib, r):
    """Fast mode at every compiled radius (tile, streaming and half-chunk
    streaming kernels) on ragged shapes — narrower / shorter than a window,
    a strip, a chunk or a band, and a batch — within the float tolerance of
    the reference; uint8 first pass bit-exact."""
    import torch

    rng = np.random.default_rng(900 + r)
    shapes = [(1, 3, 2), (1, r, 2 * r + 1), (2, 37, 300), (1, 700, 129), (3, 130, 257)]
    for shape in shapes:
        p = rng.random(shape) * 255.0
        got = ctx.iterate(torch.from_numpy(p).cuda(), r, 3, mode="fast").cpu().numpy()
        want = np.stack([oracle_lib.osbf(c, r, 3) for c in p])
        assert float(np.abs(got - want).max()) <= FLOAT_TOL * 255.0, shape
    u8 = rng.integers(0, 256, (2, 300, 290), dtype=np.uint8)
    got = ctx.iterate(torch.from_numpy(u8).cuda(), r, 1, mode="fast").cpu().numpy()
    want = np.stack([oracle_lib.osbf(c.astype(np.float64), r, 1) for c in u8])
    assert np.array_equal(bits(got), bits(want))


def test_exact_sat_bit_exact(ctx, oracle_lib):
    rng = np.random.default_rng(7)
    for h, w in [(1, 1), (3, 200), (257, 65), (300, 301)]:
        p = rng.random((h, w)) * 1000 - 500
        got = ctx.sat(torch_dev(p)).cpu().numpy()
        assert np.array_equal(bits(got), bits(oracle_lib.sat(p)))
        assert np.array_equal(bits(ctx.sat_host(p)), bits(oracle_lib.sat(p)))


def test_config_c1_full(ctx, oracle_lib):
    from paper_2108_05021_b200 import synth

    cfg = synth.CONFIGS["C1"]
    x = synth.make_input("C1")[0]
    want = oracle_lib.osbf(x, cfg.radius, cfg.iterations)
    exact = ctx.iterate(torch_dev(x), cfg.radius, cfg.iterations, mode="exact").cpu().numpy()
    assert np.array_equal(bits(exact), bits(want))
    fast = ctx.iterate(torch_dev(x), cfg.radius, cfg.iterations, mode="fast").cpu().numpy()
    assert np.abs(fast - want).max() <= FLOAT_TOL * vrange(x)


def test_config_c2_full(ctx, oracle_lib):
    from paper_2108_05021_b200 import synth

    cfg = synth.CONFIGS["C2"]
    x = synth.make_input("C2")
    want = np.stack([oracle_lib.osbf(c, cfg.radius, cfg.iterations, threads=8) for c in x])
    exact = ctx.iterate(torch_dev(x), cfg.radius, cfg.iterations, mode="exact").cpu().numpy()
    assert np.array_equal(bits(exact), bits(want))
    fast = ctx.iterate(torch_dev(x), cfg.radius, cfg.iterations, mode="fast").cpu().numpy()
    assert np.abs(fast - want).max() <= FLOAT_TOL * vrange(x)


@pytest.mark.parametrize("r", [1, 2, 4, 8, 16])
def test_config_c3_u8_radius_sweep(ctx, oracle_lib, r):
    """C3 (uint8) at 1024x1024, 10 iterations: exact mode bit-exact at every
    radius; fast mode bit-exact on the first pass (integer sums)."""
    from paper_2108_05021_b200 import synth

    x = synth.make_input("C3", shrink=4)[0]
    want = oracle_lib.osbf(x, r, 10, threads=8)
    got = ctx.iterate(torch_dev(x), r, 10, mode="exact").cpu().numpy()
    assert np.array_equal(bits(got), bits(want))
    one_fast = ctx.iterate(torch_dev(x), r, 1, mode="fast").cpu().numpy()
    assert np.array_equal(bits(one_fast), bits(oracle_lib.osbf(x, r, 1)))


@pytest.mark.parametrize("r", [1, 4, 16])
def test_config_c3_full_first_pass(ctx, oracle_lib, r):
    """Full 4096x4096 uint8: both modes bit-exact on the first pass."""
    from paper_2108_05021_b200 import synth

    x = synth.make_input("C3")[0]
    want = oracle_lib.osbf(x, r, 1, threads=8)
    for mode in ("exact", "fast"):
        got = ctx.iterate(torch_dev(x), r, 1, mode=mode).cpu().numpy()
        assert np.array_equal(bits(got), bits(want)), mode


def test_batch_equals_individual_planes(ctx):
    """C4-style batch: each plane is filtered independently (bit-identical)."""
    from paper_2108_05021_b200 import synth

    x = synth.make_input("C4", shrink=8)  # 32 x 128 x 128
    for mode in ("exact", "fast"):
        batched = ctx.iterate(torch_dev(x), 2, 4, mode=mode).cpu().numpy()
        for i in (0, 1, 17, 31):
            single = ctx.iterate(torch_dev(x[i]), 2, 4, mode=mode).cpu().numpy()
            assert np.array_equal(bits(batched[i]), bits(single))


def test_properties_at_full_size(ctx):
    """Size-independent properties on a large plane: range preservation,
    determinism, constant-plane and step fixed points, exact ~ fast."""
    import torch

    rng = np.random.default_rng(5)
    h, w = 4096, 8192
    x = torch.from_numpy(rng.random((h, w), dtype=np.float64)).cuda()
    for mode in ("exact", "fast"):
        a = ctx.iterate(x, 4, 2, mode=mode)
        b = ctx.iterate(x, 4, 2, mode=mode)
        assert torch.equal(a.view(torch.int64), b.view(torch.int64)), "not deterministic"
        assert float(a.min()) >= float(x.min()) and float(a.max()) <= float(x.max())
    e = ctx.iterate(x, 4, 2, mode="exact")
    f = ctx.iterate(x, 4, 2, mode="fast")
    assert float((e - f).abs().max()) <= FLOAT_TOL
    c = torch.full((h, w), 3.5, dtype=torch.float64, device="cuda")
    assert torch.equal(ctx.iterate(c, 16, 3, mode="exact"), c)
    assert torch.equal(ctx.iterate(c, 16, 3, mode="fast"), c)
    s = torch.where(torch.arange(w, device="cuda")[None, :] < w // 2, 0.0, 100.0).expand(h, w)
    s = s.to(torch.float64).contiguous()
    for mode in ("exact", "fast"):
        assert torch.equal(ctx.iterate(s, 8, 5, mode=mode), s)


def test_in_place_and_pitched(ctx, oracle_lib):
    import torch

    rng = np.random.default_rng(9)
    p = rng.random((64, 96)) * 10
    want = oracle_lib.osbf(p, 3, 3)
    t = torch_dev(p)
    ctx.iterate(t, 3, 3, mode="exact", out=t)  # in place
    assert np.array_equal(bits(t.cpu().numpy()), bits(want))
    big = torch.zeros((64, 128), dtype=torch.float64, device="cuda")
    big[:, :96] = torch_dev(p)
    view = big[:, :96]  # pitched input (row stride 128)
    got = ctx.iterate(view, 3, 3, mode="exact")
    assert np.array_equal(bits(got.cpu().numpy()), bits(want))


WALK_RADII = range(3, 17)  # fast radii served by the column walk (512-row blocks)


@pytest.mark.parametrize("r", [2, 7, 12])
def test_row_bands_equal_whole_image(ctx, r):
    """osbf_gpu_step_band over 128-aligned row bands (halos copied from the
    previous pass, as the multi-GPU exchange does) is bit-identical to the
    whole-image fast pass for the tile kernels; the column walk's prefix sums
    start at each band's first row, so there (bands not on its 512-row block
    grid) the bands agree to fp64 rounding (1e-9 of the range).  Unaligned
    bands stay within the float tolerance."""
    import torch

    from paper_2108_05021_b200.dist import BandLayout

    h, w, iters = 700, 300, 3
    x = torch.from_numpy(np.random.default_rng(r).random((h, w))).cuda()
    want = ctx.iterate(x, r, iters, mode="fast")
    for world in (3, 4):
        cur = x.clone()
        for _ in range(iters):
            nxt = torch.empty_like(cur)
            for rank in range(world):
                lay = BandLayout.make(h, w, r, world, rank)
                src = cur[lay.buf_row0:lay.buf_row0 + lay.buf_rows].contiguous()
                ctx.step_band(src, lay.buf_row0, nxt[lay.row0:lay.row1], lay.row0, lay.rows, h, r)
            cur = nxt
        if r in WALK_RADII:
            assert float((cur - want).abs().max()) <= 1e-9, world
        else:
            assert torch.equal(cur.view(torch.int64), want.view(torch.int64)), world
    # unaligned bands (tile grid shifted): same result within tolerance
    cur = x.clone()
    cuts = [0, 250, 333, 700]
    for _ in range(iters):
        nxt = torch.empty_like(cur)
        for r0, r1 in zip(cuts[:-1], cuts[1:]):
            b0, b1 = max(0, r0 - r), min(h, r1 + r)
            ctx.step_band(cur[b0:b1].contiguous(), b0, nxt[r0:r1], r0, r1 - r0, h, r)
        cur = nxt
    assert float((cur - want).abs().max()) <= FLOAT_TOL


@pytest.mark.parametrize("r", [3, 4, 8, 16])
def test_row_bands_walk_block_aligned_bit_identical(ctx, r):
    """Row bands whose starts sit on the column walk's 512-row block grid
    (dist.band_rows' default alignment) walk exactly the blocks of the whole
    image: bit-identical results over several passes."""
    import torch

    import paper_2108_05021_b200 as ob
    from paper_2108_05021_b200.dist import BandLayout, band_rows

    h, w, iters, world = 1536 + 77, 260, 3, 3
    assert [b[0] % 512 for b in band_rows(h, world, r)] == [0, 0, 0]
    x = torch.from_numpy(np.random.default_rng(40 + r).random((h, w))).cuda()
    ob.Context.set_fast_kernel("walk")  # a plane this small would take the tile kernels
    try:
        want = ctx.iterate(x, r, iters, mode="fast")
        assert "walk" in ctx.last_kernel
        cur = x.clone()
        for _ in range(iters):
            nxt = torch.empty_like(cur)
            for rank in range(world):
                lay = BandLayout.make(h, w, r, world, rank)
                src = cur[lay.buf_row0:lay.buf_row0 + lay.buf_rows].contiguous()
                ctx.step_band(src, lay.buf_row0, nxt[lay.row0:lay.row1], lay.row0, lay.rows, h,
                              r)
            cur = nxt
    finally:
        ob.Context.set_fast_kernel(None)
    assert torch.equal(cur.view(torch.int64), want.view(torch.int64))


@pytest.mark.parametrize("r", [2, 4, 6])
def test_row_bands_fused_push_equal_whole_image(ctx, r):
    """The fused exchange (osbf_gpu_step_band_push via dist.RowBandOSBF
    exchange='push'): every band's pass also stores its boundary rows into
    the neighbours' halo rows.  Emulated here as three ranks on one device
    (their "symmetric" buffers are local allocations, passes run one after
    another on one stream, so no kernel waits on another); the result equals
    the whole-image pass (bit-identical for the tile kernels, fp64 rounding
    for the column walk on bands off its 512-row grid)."""
    import torch

    from paper_2108_05021_b200.dist import BandLayout, RowBandOSBF

    h, w, iters, world = 700, 300, 3, 3
    x = torch.from_numpy(np.random.default_rng(10 + r).random((h, w))).cuda()
    want = ctx.iterate(x, r, iters, mode="fast")
    lays = [BandLayout.make(h, w, r, world, q) for q in range(world)]
    slot = max(q.buf_rows for q in lays) * w
    flats = [torch.full((2 * slot,), float("nan"), dtype=torch.float64, device="cuda")
             for _ in range(world)]
    ranks = [RowBandOSBF(lays[q], q, world, exchange="push", peer_buffers=lambda q: flats[q],
                         sync=lambda: None) for q in range(world)]
    for q, rb in enumerate(ranks):
        rb.prime(x[lays[q].row0:lays[q].row1])
        buf = rb._bufs[0]  # initial halos straight from the image (the emulated exchange)
        buf[:lays[q].halo_top] = x[lays[q].row0 - lays[q].halo_top:lays[q].row0]
        top = lays[q].halo_top + lays[q].rows
        buf[top:] = x[lays[q].row1:lays[q].row1 + lays[q].halo_bot]
    for it in range(iters):
        for rb in ranks:
            rb.one_pass(last=it + 1 == iters)
    got = torch.cat([rb.result() for rb in ranks])
    if r in WALK_RADII:
        assert float((got - want).abs().max()) <= 1e-9
    else:
        assert torch.equal(got.view(torch.int64), want.view(torch.int64))
    # the pushed halos hold the neighbours' final rows
    for q in range(world - 1):
        lo, hi = ranks[q], ranks[q + 1]
        top = lays[q].halo_top + lays[q].rows
        assert torch.equal(lo._bufs[lo._cur][top:], hi.result()[:r])
        assert torch.equal(hi._bufs[hi._cur][:r], lo.result()[-r:])


def test_row_band_errors(ctx):
    import torch

    import paper_2108_05021_b200 as ob

    x = torch.rand((64, 64), dtype=torch.float64, device="cuda")
    out = torch.empty_like(x)
    with pytest.raises(ob.InvalidArgument):  # exact mode cannot be banded
        ctx.step_band(x, 0, out, 0, 64, 64, 2, mode="exact")
    with pytest.raises(ob.OutOfRange):  # halo missing
        ctx.step_band(x[8:], 8, out[8:32], 8, 24, 64, 2)


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("r", [1, 2, 3, 4])
def test_temporal_blocking_matches_single_passes(oracle_lib, r, k):
    """k passes per launch (tile staged with a k*r halo, intermediates in
    shared memory, zero outside the image, clipped counts at the global
    border) = k single passes; a remainder runs as a shorter launch."""
    import paper_2108_05021_b200 as ob

    ctxk = ob.Context(0)
    ctxk.set_temporal_blocking(k)
    rng = np.random.default_rng(40 + r + 10 * k)
    for h, w, it in [(300, 250, 5), (64, 64, 2), (130, 67, 4), (5, 3, 3), (200, 128, 7)]:
        p = rng.random((h, w)) * 100.0
        single = ob.default_context().iterate(torch_dev(p), r, it, mode="fast").cpu().numpy()
        before = ctxk.launches
        tb = ctxk.iterate(torch_dev(p), r, it, mode="fast").cpu().numpy()
        # TMA needs 16-byte row pitch: odd widths fall back to single passes
        if w % 2 == 0:
            assert ctxk.launches - before == -(-it // k)
            assert ctxk.last_kernel in ("fast_tma_stepk", "fast_tma_step", "fast_walk_step")
        else:
            assert ctxk.launches - before == it
        assert np.abs(tb - single).max() <= 1e-9 * 100.0
        assert np.abs(tb - oracle_lib.osbf(p, r, it)).max() <= FLOAT_TOL * vrange(p)
    # uint8: the first pass inside the launch divides exactly (bit-exact);
    # after it, exact ties between windows are common and the
    # multi-pass tiles sum in another order than single passes, so only
    # near-tie pixels may differ
    u8 = rng.integers(0, 256, (96, 100), dtype=np.uint8)
    tb = ctxk.iterate(torch_dev(u8), r, k, mode="fast").cpu().numpy()
    single = ob.default_context().iterate(torch_dev(u8), r, k, mode="fast").cpu().numpy()
    assert np.mean(np.abs(tb - single) > 1e-9 * 255.0) < 0.02
    ctxk.iterate(torch_dev(u8), r, 1, mode="fast")  # one pass: single kernel, exact
    ctxk.close()


@pytest.mark.parametrize("shape", [(200, 180), (100, 40, 96)])
def test_exact_non_finite_samples_bit_exact(ctx, oracle_lib, shape):
    """NaN / inf samples propagate through the reference's table exactly as
    its serial adds do; exact mode (table path for a lone plane, the strip
    walk for batches) matches the oracle bit for bit, NaN positions
    included.  Also raises the table-range flag, after which the stencil
    keeps its guarded division."""
    import torch

    rng = np.random.default_rng(77)
    p = rng.random(shape) * 50.0
    flat = p.reshape(-1)
    flat[rng.integers(0, flat.size, 5)] = np.nan
    flat[rng.integers(0, flat.size, 3)] = np.inf
    flat[rng.integers(0, flat.size, 2)] = -np.inf
    got = ctx.iterate(torch.from_numpy(p).cuda(), 3, 2, mode="exact").cpu().numpy()
    planes = p.reshape((-1,) + p.shape[-2:])
    want = np.stack([oracle_lib.osbf(c, 3, 2) for c in planes]).reshape(p.shape)
    assert np.array_equal(bits(got), bits(want))
