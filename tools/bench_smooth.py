"""End-to-end timing of the `osbf smooth` edge (osbf_gpu_smooth_raster_host:
uint8/uint16 raster in, quantised raster out, promotion + quantisation on the
GPU) against the fp64 host path a reference-style caller would take
(read_image's promoted planes through osbf_gpu_filter_multichannel_host, then
quantise on the host).  Wall clock around the host-synchronous calls, median
of --reps after a warm-up.
usage: python tools/bench_smooth.py [--size 4096] [--iters 10] [--reps 5]"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_05021_b200 as ob

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=4096)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
ctx = ob.Context(0)
rng = np.random.default_rng(5)


def timed(fn):
    fn()
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return sorted(ts)[len(ts) // 2]


for channels, filt, r in ((3, "osbf", 2), (1, "osbf", 2), (3, "fast-osbf", 2), (3, "box", 2),
                          (3, "osbf", 8)):
    shape = (a.size, a.size, 3) if channels == 3 else (a.size, a.size)
    x = (rng.random(shape) * 256).astype(np.uint8)
    t_raster = timed(lambda: ctx.smooth_raster(x, filt, r, a.iters))
    planes = [np.ascontiguousarray(x[..., c] if channels == 3 else x, dtype=np.float64)
              for c in range(channels)]
    variant = {"osbf": ob.FilterVariant.OsbfExact, "fast-osbf": ob.FilterVariant.OsbfFast,
               "box": ob.FilterVariant.Box}[filt]

    def f64_path():
        outs = ctx.filter_multichannel_host(planes, r, a.iters, variant=variant)
        return [np.clip(np.floor(o + 0.5), 0, 255).astype(np.uint8) for o in outs]

    t_f64 = timed(f64_path)
    px_iter = a.size * a.size * channels * a.iters
    print(json.dumps({"raster": list(shape), "filter": filt, "r": r, "iters": a.iters,
                      "smooth_raster_ms": round(t_raster * 1e3, 2),
                      "smooth_raster_Mpx_iter_s": round(px_iter / t_raster / 1e6, 1),
                      "pcie_bytes": 2 * x.nbytes,
                      "f64_host_path_ms": round(t_f64 * 1e3, 2),
                      "f64_pcie_bytes": 2 * 8 * x.size,
                      "speedup": round(t_f64 / t_raster, 2)}))
