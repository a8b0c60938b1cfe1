"""Per-pass timing of the OSBF kernels (CUDA events, warm, L2-flushed), with
the SM clocks sampled during the timed passes (nvidia-smi, bench.py's
ClockSampler) so every record carries its clock evidence.
usage: python tools/prof_pass.py [--mode fast|exact|fastosbf|box|osbf3d|box3d] [--radii 1,2,4,8,16]
                                 [--shape B,H,W] [--dtype f64|f32|u8]
(fastosbf = paper Algorithm 3, osbf_gpu_fast_osbf; box = osbf_gpu_box_filter;
 osbf3d / box3d = the 3-D filters with --shape read as D,H,W)"""
import argparse, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2108_05021_b200 as ob
from bench import ClockSampler

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="fast")
ap.add_argument("--radii", default="1,2,4,8,16")
ap.add_argument("--shape", default="256,1024,1024")
ap.add_argument("--dtype", default="f64")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--tag", default="")
ap.add_argument("--iters", type=int, default=1, help="passes per timed call (temporal blocking needs >= 2)")
a = ap.parse_args()
B, H, W = map(int, a.shape.split(","))
ctx = ob.Context(0)
if a.dtype == "u8":
    x = torch.randint(0, 256, (B, H, W), dtype=torch.uint8, device="cuda")
else:
    x = torch.rand((B, H, W), dtype=torch.float64, device="cuda").to(
        {"f64": torch.float64, "f32": torch.float32}[a.dtype])
y = torch.empty((B, H, W), dtype=torch.float64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
in_b = {"f64": 8, "f32": 4, "u8": 1}[a.dtype]
for r in map(int, a.radii.split(",")):
    run = {"fastosbf": lambda: ctx.fast_osbf(x, r, 1, out=y),
           "box": lambda: ctx.box_filter(x, r, 1, out=y),
           "osbf3d": lambda: ctx.osbf_3d(x, r, 1, out=y),
           "box3d": lambda: ctx.box_filter_3d(x, r, 1, out=y)}.get(
               a.mode, lambda: ctx.iterate(x, r, a.iters, mode=a.mode, out=y))
    for _ in range(3):
        run()
    kernel = ctx.last_kernel
    torch.cuda.synchronize()
    s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(); run(); e0.record(); torch.cuda.synchronize()
    reps = max(a.reps, int(800.0 / max(s0.elapsed_time(e0), 1e-3)))  # >= ~0.8 s sampled
    clk = ClockSampler(0)
    clk.start()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); run(); e.record()
        torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    c = clk.stop()
    ts.sort(); ms = ts[len(ts) // 2] / a.iters
    px = B * H * W
    gbs = px * ((in_b + 8) + (a.iters - 1) * 16) / a.iters / (ms / 1e3) / 1e9
    print(json.dumps({"mode": a.mode, "tag": a.tag, "kernel": kernel, "r": r, "shape": [B, H, W],
                      "dtype": a.dtype, "ms_per_pass": round(ms, 4),
                      "gpx_per_s": round(px / ms / 1e6, 2), "alg_GBps": round(gbs, 1),
                      "frac_of_peak": round(gbs / peak, 3),
                      "clocks": {"sm_mhz": c.get("sm_mhz"), "reasons": c.get("reasons")}}), flush=True)
