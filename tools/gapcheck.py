"""Per-pass time inside a multi-pass iterate() vs isolated passes (launch-gap check)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_05021_b200 as ob
ctx = ob.Context(0)
B, H, W = 256, 1024, 1024
x = torch.rand((B, H, W), dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, reps=5):
    ts = []
    for _ in range(reps):
        flush.fill_(1); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return sorted(ts)[len(ts)//2]
for _ in range(2): ctx.iterate(x, 2, 20, mode="fast", out=y)
one = t(lambda: ctx.iterate(x, 2, 1, mode="fast", out=y))
twenty = t(lambda: ctx.iterate(x, 2, 20, mode="fast", out=y))
# host-side cost of enqueueing 20 passes
import time
torch.cuda.synchronize(); t0 = time.perf_counter(); ctx.iterate(x, 2, 20, mode="fast", out=y); t1 = time.perf_counter(); torch.cuda.synchronize()
print(json.dumps({"one_pass_ms": one, "twenty_pass_ms": twenty, "per_pass_in_20": twenty / 20, "host_enqueue_20_ms": (t1 - t0) * 1e3}))
