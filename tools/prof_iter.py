"""Per-iteration timing of multi-pass iterate() (fast mode), for temporal-blocking A/B."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_05021_b200 as ob
ctx = ob.Context(0)
B, H, W = map(int, (sys.argv[1] if len(sys.argv) > 1 else "256,1024,1024").split(","))
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
radii = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "1,2").split(",")]
x = torch.rand((B, H, W), dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for r in radii:
    for _ in range(2): ctx.iterate(x, r, iters, mode="fast", out=y)
    ts = []
    for _ in range(5):
        flush.fill_(1); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); ctx.iterate(x, r, iters, mode="fast", out=y); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ms = sorted(ts)[2]
    print(json.dumps({"tb2": os.environ.get("OSBF_GPU_TB2", "1"), "r": r, "iters": iters,
                      "ms": round(ms, 3), "gpx_iter_per_s": round(B * H * W * iters / ms / 1e6, 1)}))
