"""Per-pass device time across a long run of back-to-back single passes (clock/power drift check)."""
import sys, os, json, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_05021_b200 as ob
ctx = ob.Context(0)
x = torch.rand((256, 1024, 1024), dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "50"], stdout=open("/tmp/trace_clk.csv", "w"))
torch.cuda.synchronize()
ev[0].record()
a, b = x, y
for i in range(n):
    ctx.iterate(a, 2, 1, mode="fast", out=b)
    ev[i + 1].record()
    a, b = b, a
torch.cuda.synchronize()
smi.terminate(); smi.wait()
t = [ev[i].elapsed_time(ev[i + 1]) for i in range(n)]
clk = [l.strip() for l in open("/tmp/trace_clk.csv")]
print(json.dumps({"first10": [round(v, 3) for v in t[:10]], "last10": [round(v, 3) for v in t[-10:]],
                  "median": sorted(t)[n // 2]}))
print("clocks:", clk[:3], "...", clk[-3:])
