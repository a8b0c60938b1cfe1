"""Reference-interface behaviour of the Python mirror on the GPU: error
types, zero-iteration quirk, multichannel semantics (filters2d.hpp:371-400)."""
import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu


def test_error_behaviour_matches_reference():
    import paper_2108_05021_b200 as ob

    p = np.random.default_rng(1).random((8, 8))
    with pytest.raises(ob.InvalidArgument):
        ob.osbf_step(p, 0)  # filters2d.hpp:62-63
    with pytest.raises(ob.InvalidArgument):
        ob.osbf(p, 0, 1)
    with pytest.raises(ob.InvalidArgument):
        ob.osbf(p, 2, -1)  # filters2d.hpp:92-93
    # iterations == 0 copies without validating r (filters2d.hpp:94-97)
    assert np.array_equal(ob.osbf(p, 0, 0), p)
    assert np.array_equal(ob.osbf(p, -5, 0), p)
    with pytest.raises(ob.InvalidArgument):
        ob.osbf(np.zeros((0, 4)), 2, 1)  # core.hpp:20-21
    ctx = ob.default_context()
    st = ctx._lib.osbf_gpu_osbf_step_host(ctx.handle, None, None, 4, 4, 0, 0)
    assert st == 1 and b"radius must be >= 1" in ctx._lib.osbf_gpu_last_error()


def test_multichannel_semantics():
    import paper_2108_05021_b200 as ob

    cfg = ob.FilterConfig(radius=2, iterations=2)
    flat = [np.full((12, 12), v) for v in (1.0, 2.0, 3.0)]
    out = ob.filter_multichannel(flat, cfg)
    for o, c in zip(out, flat):
        assert np.array_equal(o, c)
    rng = np.random.default_rng(2)
    rgb = [rng.random((12, 12)) * 255 for _ in range(3)]
    filtered = ob.filter_multichannel(rgb, cfg)
    for f, c in zip(filtered, rgb):
        assert np.array_equal(bits(f), bits(ob.osbf(c, 2, 2)))
    with pytest.raises(ob.InvalidArgument):
        ob.filter_multichannel(rgb, ob.FilterConfig(radius=0))
    with pytest.raises(ob.InvalidArgument):
        ob.filter_multichannel(rgb * 2, cfg)  # 6 channels
    with pytest.raises(ob.InvalidArgument):  # not on the GPU path
        ob.filter_multichannel(rgb, ob.FilterConfig(variant=ob.FilterVariant.Gaussian))
    boxed = ob.filter_multichannel(rgb, ob.FilterConfig(radius=2, iterations=2,
                                                        variant=ob.FilterVariant.Box))
    for f, c in zip(boxed, rgb):
        assert np.array_equal(bits(f), bits(ob.box_filter(c, 2, 2)))


def test_launch_counter_counts_kernels(ctx):
    import torch

    x = torch.rand((64, 64), dtype=torch.float64, device="cuda")
    before = ctx.launches
    ctx.iterate(x, 2, 3, mode="exact")
    # the whole-table path: 3 kernels per exact pass (row carries, strip
    # table builder, stencil walk)
    assert ctx.launches - before == 9 and "exact_table_strip" in ctx.last_kernel
    xb = torch.rand((300, 64, 64), dtype=torch.float64, device="cuda")
    import paper_2108_05021_b200 as ob

    ob.Context.set_exact_kernel("strip")
    try:
        before = ctx.launches
        ctx.iterate(xb, 2, 3, mode="exact")
        # the fused strip walk: 2 kernels per pass (row carries + strip)
        assert ctx.launches - before == 6 and "exact_strip" in ctx.last_kernel
    finally:
        ob.Context.set_exact_kernel(None)
    before = ctx.launches
    ctx.iterate(x, 2, 3, mode="fast")
    assert ctx.launches - before == 3


def test_dtype_promotion_is_exact(ctx, oracle_lib):
    import torch

    rng = np.random.default_rng(4)
    u8 = rng.integers(0, 256, (33, 45), dtype=np.uint8)
    f32 = (rng.random((33, 45)) * 3).astype(np.float32)
    for a in (u8, f32):
        got = ctx.iterate(torch.from_numpy(a).cuda(), 2, 2, mode="exact").cpu().numpy()
        assert np.array_equal(bits(got), bits(oracle_lib.osbf(a.astype(np.float64), 2, 2)))


@pytest.mark.parametrize("mode,r", [("fast", 2), ("fast", 6), ("exact", 3)])
def test_host_batch_pipeline_matches_device_path(ctx, mode, r):
    """Host-buffer batches >= 64 MB go through in overlapped chunks (upload /
    passes / download on three streams); the result is bit-identical to one
    device-resident launch over the whole batch."""
    import torch

    rng = np.random.default_rng(r)
    x = (rng.random((9, 1024, 1024)) * 255).astype(np.float32)  # 72 MB of fp64 output
    got = ctx.osbf_host(x, r, 2, mode=mode)
    want = ctx.iterate(torch.from_numpy(x).cuda(), r, 2, mode=mode).cpu().numpy()
    assert np.array_equal(got.view(np.int64), want.view(np.int64))


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_repeated_calls_replay_a_graph(ctx, oracle_lib, mode):
    """A repeated call with the same buffers is replayed as one CUDA graph
    (captured on the second call): results follow the CURRENT input contents,
    and the launch counter still counts the kernels inside the graph."""
    import torch

    x = torch.rand((3, 96, 80), dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    before = ctx.launches
    ctx.iterate(x, 2, 4, mode=mode, out=y)
    per_call = ctx.launches - before
    for _ in range(3):  # plain, capture, replay, replay
        ctx.iterate(x, 2, 4, mode=mode, out=y)
    assert ctx.launches - before == 4 * per_call
    x.copy_(torch.rand_like(x) * 255)  # new contents, same buffers -> replay
    ctx.iterate(x, 2, 4, mode=mode, out=y)
    got = y.cpu().numpy()
    for b in range(3):
        want = oracle_lib.osbf(x[b].cpu().numpy(), 2, 4)
        if mode == "exact":
            assert np.array_equal(bits(got[b]), bits(want))
        else:
            assert np.abs(got[b] - want).max() <= 1e-9 * 255
    z = torch.empty_like(x)  # a different output buffer is a different graph key
    ctx.iterate(x, 2, 4, mode=mode, out=z)
    assert torch.equal(z, y)


def test_fast_mode_beyond_generic_radius_runs_exact_kernels(ctx, oracle_lib):
    """The reference accepts any r; fast mode has kernels up to
    Context.fast_max_radius() (templated to 16, then the generic walk) and
    runs larger windows on the exact kernels (bit-identical)."""
    import torch

    import paper_2108_05021_b200 as ob

    r = ob.Context.fast_max_radius() + 3
    p = np.random.default_rng(3).random((90, 2 * r + 7)) * 255
    got = ctx.iterate(torch.from_numpy(p).cuda(), r, 2, mode="fast").cpu().numpy()
    assert np.array_equal(bits(got), bits(oracle_lib.osbf(p, r, 2)))


def test_out_argument_is_validated(ctx):
    """A caller-supplied ``out`` must be float64, on the input's device, of
    the input's shape, with contiguous rows (no silent 8-byte writes into a
    smaller buffer)."""
    import torch

    import paper_2108_05021_b200 as ob

    x = torch.rand((2, 40, 48), dtype=torch.float64, device="cuda")
    for bad in (torch.empty((2, 40, 48), dtype=torch.float32, device="cuda"),
                torch.empty((2, 40, 47), dtype=torch.float64, device="cuda"),
                torch.empty((2, 48, 40), dtype=torch.float64, device="cuda"),
                torch.empty((2, 40, 96), dtype=torch.float64, device="cuda")[:, :, ::2],
                torch.empty((2, 40, 48), dtype=torch.float64)):
        for fn in (lambda o: ctx.iterate(x, 2, 1, mode="fast", out=o),
                   lambda o: ctx.box_filter(x, 2, 1, out=o),
                   lambda o: ctx.fast_osbf(x, 2, 1, out=o)):
            with pytest.raises(ob.InvalidArgument):
                fn(bad)
    good = torch.empty((2, 40, 48), dtype=torch.float64, device="cuda")
    ctx.iterate(x, 2, 1, mode="fast", out=good)
    vol = torch.rand((6, 7, 8), dtype=torch.float64, device="cuda")
    with pytest.raises(ob.InvalidArgument):
        ctx.osbf_3d(vol, 1, 1, out=torch.empty((6, 7, 9), dtype=torch.float64, device="cuda"))
    band_src = torch.rand((30, 48), dtype=torch.float64, device="cuda")
    with pytest.raises(ob.InvalidArgument):  # out smaller than out_rows
        ctx.step_band(band_src, 0, torch.empty((10, 48), dtype=torch.float64, device="cuda"),
                      0, 20, 30, 2)


def test_calls_on_different_streams_are_ordered(ctx, oracle_lib):
    """Calls issued on different streams share the context's scratch; the
    context orders them, so alternating streams gives the same results as
    one stream."""
    import torch

    rng = np.random.default_rng(3)
    planes = [rng.random((300, 500)) for _ in range(4)]
    want = [oracle_lib.osbf(p, 3, 4) for p in planes]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    xs = [torch.from_numpy(p).cuda() for p in planes]
    torch.cuda.synchronize()
    outs = []
    for i, x in enumerate(xs):
        with torch.cuda.stream(streams[i % 2]):
            outs.append(ctx.iterate(x, 3, 4, mode="exact"))
    torch.cuda.synchronize()
    for o, w in zip(outs, want):
        assert np.array_equal(bits(o.cpu().numpy()), bits(w))


@pytest.mark.parametrize("w", [301, 77])
def test_band_pass_odd_width_unaligned_cuts(ctx, oracle_lib, w):
    """Row bands on layouts TMA cannot describe (odd fp64 widths: the
    two-phase tile kernel) with unaligned cuts: the last partial tile of a
    band must not read past the caller's band buffer, and the result equals
    the whole-image pass."""
    import torch

    r, H = 3, 203
    p = torch.from_numpy(np.random.default_rng(w).random((H, w))).cuda()
    whole = ctx.iterate(p, r, 1, mode="fast")
    out = torch.empty((H, w), dtype=torch.float64, device="cuda")
    for a, b in ((0, 61), (61, 130), (130, H)):
        i0, i1 = max(0, a - r), min(H, b + r)
        src = p[i0:i1].clone()  # a tight buffer: nothing past its last row
        ctx.step_band(src, i0, out[a:b], a, b - a, H, r)
    assert float((out - whole).abs().max()) <= 1e-9


def test_batch_above_grid_limit_is_rejected(ctx):
    """Planes ride in gridDim.z: a batch above 65535 is refused up front
    (InvalidArgument), not failed at launch."""
    import torch

    import paper_2108_05021_b200 as ob

    x = torch.rand((65536, 2, 2), dtype=torch.float64, device="cuda")
    with pytest.raises(ob.InvalidArgument):
        ctx.iterate(x, 1, 1, mode="fast")
