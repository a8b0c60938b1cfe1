"""Run a few fast/exact passes of one configuration (for ncu captures):
python tools/run_passes.py --r 4 --shape 256,1024,1024 --mode fast --passes 3"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_05021_b200 as ob

ap = argparse.ArgumentParser()
ap.add_argument("--r", type=int, default=4)
ap.add_argument("--shape", default="256,1024,1024")
ap.add_argument("--mode", default="fast")
ap.add_argument("--passes", type=int, default=3)
ap.add_argument("--dtype", default="f64")
a = ap.parse_args()
B, H, W = map(int, a.shape.split(","))
ctx = ob.Context(0)
x = torch.rand((B, H, W), dtype=torch.float64, device="cuda")
if a.dtype == "f32":
    x = x.float()
y = torch.empty((B, H, W), dtype=torch.float64, device="cuda")
for _ in range(a.passes):
    ctx.iterate(x, a.r, 1, mode=a.mode, out=y)
torch.cuda.synchronize()
print("ok", ctx.last_kernel)
