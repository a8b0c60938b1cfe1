"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

The reference repository ships no golden files — its tests generate every
input from seeds (proj/tests/support/fixtures.hpp:15-71).  This script runs
the reference itself (its headers compiled behind oracle/ref_shim.cpp) on
seeded inputs and stores inputs + outputs, so the C restatement and the GPU
path can be pinned against real reference outputs on machines where the
reference tree is absent (the GPU box).

    python tests/golden/make_golden.py          # rewrites the .npz files

Cases mirror the reference's own hot-path tests (file:line under
/root/reference/proj/tests/) plus the BASELINE configs at reduced size.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from oracle import Reference  # noqa: E402
from paper_2108_05021_b200 import synth  # noqa: E402


def random_plane(h, w, seed, lo=0.0, hi=255.0):
    rng = np.random.default_rng(seed)
    return lo + (hi - lo) * rng.random((h, w))


def checkerboard(w, h, cell, lo, hi):
    y, x = np.mgrid[0:h, 0:w]
    return np.where(((x // cell + y // cell) % 2) == 0, lo, hi).astype(np.float64)


def step(w, h, edge, lo, hi):
    x = np.arange(w)[None, :].repeat(h, 0)
    return np.where(x < edge, lo, hi).astype(np.float64)


def cases():
    """(name, input (H,W) or (C,H,W), r, iterations)."""
    out = []
    # test_filters2d.cpp:142-147 — osbf vs brute force, 24x24, r in {1,2,3,5}, 3 iterations
    for r in (1, 2, 3, 5):
        out.append((f"random24_r{r}", random_plane(24, 24, 200 + r), r, 3))
    # acceptance.cpp:137-152 — 64x64 planes, r in {1,2,3,5}, 3 iterations (2 of the 50)
    for k in (0, 1):
        for r in (1, 2, 3, 5):
            out.append((f"random64_k{k}_r{r}", random_plane(64, 64, 1000 + k), r, 3))
    # C3-style uint8 mosaic, radius sweep, 10 iterations (bit-exact target)
    rng = np.random.default_rng(33)
    u8 = synth.u8_mosaic(96, 80, rng, block=(4, 40))
    for r in (1, 2, 4, 8, 16):
        out.append((f"u8mosaic_r{r}", u8, r, 10))
    # BASELINE C1 / C2 at reduced size (float32 inputs)
    out.append(("c1_shrink4", synth.make_input("C1", shrink=4)[0], 2, 10))
    out.append(("c2_shrink12", synth.make_input("C2", shrink=12), 3, 30))
    # edge cases: degenerate shapes, windows wider than the image, fixed points
    out.append(("one_px", np.array([[7.5]]), 2, 3))
    out.append(("row_1x17", random_plane(1, 17, 5), 3, 2))
    out.append(("col_13x1", random_plane(13, 1, 6), 2, 2))
    out.append(("tiny_7x5_r16", random_plane(7, 5, 7), 16, 4))
    out.append(("ragged_37x29_r4", random_plane(37, 29, 8), 4, 3))
    out.append(("constant_9x9", np.full((9, 9), 3.5), 2, 1))
    out.append(("step_32x16_r5", step(32, 16, 16, 0.0, 100.0), 5, 1))
    out.append(("step_64x32_30it", step(64, 32, 32, 0.0, 100.0), 2, 30))
    out.append(("checker_64_cell9_r3", checkerboard(64, 64, 9, 10.0, 200.0), 3, 1))
    out.append(("checker_32_cell4_r3", checkerboard(32, 32, 4, 0.0, 255.0), 3, 1))
    out.append(("zero_iters", random_plane(10, 10, 3), 2, 0))
    out.append(("negative_values", random_plane(20, 20, 9, -1e3, 1e3), 2, 4))
    return out


def fast_osbf_cases():
    """(name, input, r, iterations) for fast_osbf (filters2d.hpp:105-154)."""
    out = []
    # test_filters2d.cpp:169-177 — constant plane and ideal steps are fixed points
    out.append(("constant_9x9_r3", np.full((9, 9), 11.0), 3, 2))
    for r in (1, 2, 5):
        out.append((f"step_32x16_r{r}", step(32, 16, 16, 0.0, 100.0), r, 1))
    # test_filters2d.cpp:179-186 / acceptance.cpp:106-134 — a structured image
    # (seeded mosaic + noise stands in for the reference's phantom fixture)
    ph = synth.make_input("C1", shrink=4)[0].astype(np.float64) * 255.0
    for r in (2, 6):
        out.append((f"mosaic128_r{r}", ph, r, 10))
    for r in (1, 3, 7, 16):
        out.append((f"random_50x37_r{r}", random_plane(37, 50, 300 + r), r, 4))
    rng = np.random.default_rng(34)
    out.append(("u8mosaic_r4", synth.u8_mosaic(96, 80, rng, block=(4, 40)), 4, 10))
    out.append(("one_px", np.array([[7.5]]), 2, 3))
    out.append(("row_1x17", random_plane(1, 17, 15), 3, 2))
    out.append(("col_13x1", random_plane(13, 1, 16), 2, 2))
    out.append(("zero_iters", random_plane(10, 10, 13), 2, 0))
    out.append(("c2_shrink12", synth.make_input("C2", shrink=12), 3, 5))
    return out


def box_filter_cases():
    """(name, input, r, iterations) for box_filter (filters2d.hpp:38-56)."""
    out = []
    # test_filters2d.cpp:44-48 — constant planes are fixed points
    for r in (1, 3):
        out.append((f"constant_11x7_r{r}", np.full((7, 11), 42.0), r, 3))
    # test_filters2d.cpp:50-69 — against the brute-force oracle, several radii
    for r in (1, 2, 4, 9, 16):
        out.append((f"random_45x31_r{r}", random_plane(31, 45, 500 + r), r, 3))
    rng = np.random.default_rng(35)
    out.append(("u8mosaic_r2", synth.u8_mosaic(96, 80, rng, block=(4, 40)), 2, 5))
    out.append(("one_px", np.array([[7.5]]), 2, 3))
    out.append(("row_1x17", random_plane(1, 17, 25), 3, 2))
    out.append(("zero_iters", random_plane(10, 10, 23), 2, 0))
    out.append(("c2_shrink12", synth.make_input("C2", shrink=12), 3, 2))
    return out


def filter3d_cases():
    """(name, volume (D, H, W), r, iterations, osbf3) for filters3d.hpp."""
    out = []
    rng = np.random.default_rng(36)
    for r in (1, 2, 3):
        out.append((f"osbf3d_random_9x10x12_r{r}", rng.random((9, 10, 12)) * 255, r, 2, True))
    step = np.where(np.arange(16)[None, None, :] < 8, 10.0, 90.0) * np.ones((8, 6, 1))
    out.append(("osbf3d_step_8x6x16_r2", step, 2, 1, True))  # test_filters3d.cpp:80-100
    out.append(("osbf3d_ragged_5x1x7_r2", rng.random((5, 1, 7)), 2, 3, True))
    for r in (1, 3):
        out.append((f"box3d_random_7x9x11_r{r}", rng.random((7, 9, 11)) * 100, r, 2, False))
    out.append(("box3d_constant_r2", np.full((4, 5, 6), 2.5), 2, 3, False))
    return out


def smooth_cases():
    """(name, raster, filter, r, iterations) for the `osbf smooth` edge
    (tools/osbf_main.cpp:63-83), run through the reference's own file I/O."""
    rng = np.random.default_rng(37)
    step = np.where(np.arange(64)[None, :] < 32, 0, 100).astype(np.uint8) * np.ones((64, 1), np.uint8)
    board = ((np.arange(48)[:, None] // 6 + np.arange(40)[None, :] // 6) % 2 * 255).astype(np.uint8)
    return [
        ("step_64_osbf_r2_it10", step, "osbf", 2, 10),  # test_cli.cpp:97-106
        ("board_box_it0", board, "box", 2, 0),  # test_cli.cpp:108-114
        ("rgb_u8_osbf_r2", (rng.random((37, 29, 3)) * 256).astype(np.uint8), "osbf", 2, 3),
        ("rgb_u8_fast_r3", (rng.random((23, 41, 3)) * 256).astype(np.uint8), "fast-osbf", 3, 2),
        ("rgb_u8_box_r1", (rng.random((19, 17, 3)) * 256).astype(np.uint8), "box", 1, 4),
        ("gray_u16_osbf_r4", (rng.random((33, 35)) * 65536).astype(np.uint16), "osbf", 4, 2),
        ("gray_u16_box_r2", (rng.random((9, 70)) * 65536).astype(np.uint16), "box", 2, 1),
        ("row_u8_osbf_r3", (rng.random((1, 50)) * 256).astype(np.uint8), "osbf", 3, 2),
    ]


def main() -> None:
    ref = Reference()
    ref.set_max_threads(1)
    for name, inp, r, iters in cases():
        if inp.ndim == 3:
            out = ref.filter_multichannel(inp.astype(np.float64), r, iters)
            means, sel = ref.subwindow_means(inp[0].astype(np.float64), r)
        else:
            out = ref.osbf(inp.astype(np.float64), r, iters)
            means, sel = ref.subwindow_means(inp.astype(np.float64), r)
        extra = {"step1_means": means} if means.shape[0] * means.shape[1] <= 1024 else {}
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), input=inp, output=out,
                            radius=r, iterations=iters, step1_sel=sel, **extra)
        print(f"{name:24s} in {inp.shape} {inp.dtype} r={r} it={iters}")
    os.makedirs(os.path.join(HERE, "fastosbf"), exist_ok=True)
    for name, inp, r, iters in fast_osbf_cases():
        x = inp.astype(np.float64)
        out = (ref.filter_multichannel(x, r, iters, variant="fast") if x.ndim == 3
               else ref.fast_osbf(x, r, iters))
        np.savez_compressed(os.path.join(HERE, "fastosbf", f"{name}.npz"), input=inp, output=out,
                            radius=r, iterations=iters)
        print(f"fastosbf/{name:20s} in {inp.shape} {inp.dtype} r={r} it={iters}")
    os.makedirs(os.path.join(HERE, "boxfilter"), exist_ok=True)
    for name, inp, r, iters in box_filter_cases():
        x = inp.astype(np.float64)
        out = (np.stack([ref.box_filter(c, r, iters) for c in x]) if x.ndim == 3
               else ref.box_filter(x, r, iters))
        np.savez_compressed(os.path.join(HERE, "boxfilter", f"{name}.npz"), input=inp,
                            output=out, radius=r, iterations=iters)
        print(f"boxfilter/{name:20s} in {inp.shape} {inp.dtype} r={r} it={iters}")
    os.makedirs(os.path.join(HERE, "filters3d"), exist_ok=True)
    for name, vol, r, iters, osbf3 in filter3d_cases():
        out = ref.osbf_3d(vol, r, iters) if osbf3 else ref.box_filter_3d(vol, r, iters)
        np.savez_compressed(os.path.join(HERE, "filters3d", f"{name}.npz"), input=vol,
                            output=out, radius=r, iterations=iters, osbf3=osbf3,
                            svt=ref.svt(vol))
        print(f"filters3d/{name:28s} {vol.shape} r={r} it={iters}")
    os.makedirs(os.path.join(HERE, "smooth"), exist_ok=True)
    import tempfile

    with tempfile.TemporaryDirectory() as tmp:
        for name, raster, filt, r, iters in smooth_cases():
            out = ref.smooth_raster(raster, filt, r, iters, tmp)
            np.savez_compressed(os.path.join(HERE, "smooth", f"{name}.npz"), input=raster,
                                output=out, filter=filt, radius=r, iterations=iters)
            print(f"smooth/{name:24s} {raster.shape} {raster.dtype} {filt} r={r} it={iters}")
    # integral.hpp / test_integral.cpp:19-29 known SAT
    p = np.array([[1.0, 2.0], [3.0, 4.0]])
    np.savez_compressed(os.path.join(HERE, "sat_2x2.npz"), input=p, cumsum=ref.sat(p))


if __name__ == "__main__":
    main()
