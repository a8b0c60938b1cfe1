"""Quick per-pass timing of the OSBF kernels (CUDA events, warm, L2-flushed).
usage: python tools/prof_pass.py [--mode fast|exact|fastosbf|box|osbf3d|box3d] [--radii 1,2,4,8,16]
                                 [--shape B,H,W]
(fastosbf = paper Algorithm 3, osbf_gpu_fast_osbf; box = osbf_gpu_box_filter;
 osbf3d / box3d = the 3-D filters with --shape read as D,H,W)"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_05021_b200 as ob

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="fast")
ap.add_argument("--radii", default="1,2,4,8,16")
ap.add_argument("--shape", default="256,1024,1024")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
B, H, W = map(int, a.shape.split(","))
ctx = ob.Context(0)
x = torch.rand((B, H, W), dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
for r in map(int, a.radii.split(",")):
    run = {"fastosbf": lambda: ctx.fast_osbf(x, r, 1, out=y),
           "box": lambda: ctx.box_filter(x, r, 1, out=y),
           "osbf3d": lambda: ctx.osbf_3d(x, r, 1, out=y),
           "box3d": lambda: ctx.box_filter_3d(x, r, 1, out=y)}.get(
               a.mode, lambda: ctx.iterate(x, r, 1, mode=a.mode, out=y))
    for _ in range(3):
        run()
    ts = []
    for _ in range(a.reps):
        flush.fill_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); run(); e.record()
        torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort(); ms = ts[len(ts) // 2]
    px = B * H * W
    gbs = px * 16 / (ms / 1e3) / 1e9
    print(json.dumps({"mode": a.mode, "r": r, "shape": [B, H, W], "ms_per_pass": round(ms, 4),
                      "gpx_per_s": round(px / ms / 1e6, 2), "alg_GBps": round(gbs, 1),
                      "frac_of_peak": round(gbs / peak, 3)}))
