"""Random-shape fuzz of the default exact path (row carries + strip table
builder + generic stencil walk) against the oracle: bit-identical or report."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2108_05021_b200 as ob
import oracle

orc = oracle.Oracle()
ctx = ob.Context(0)
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
bad = 0
n = int(sys.argv[2]) if len(sys.argv) > 2 else 80
for i in range(n):
    b = int(rng.choice([1, 1, 2, 3, 7]))
    h = int(rng.integers(1, 400)); w = int(rng.integers(1, 400))
    if rng.random() < 0.3: w = int(rng.choice([31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256, 257]))
    if rng.random() < 0.3: h = int(rng.choice([1, 2, 31, 32, 33, 63, 64, 65, 96, 128, 129]))
    r = int(rng.choice([1, 2, 3, 5, 8, 13, 16, 17, 23, 32, 47, 62, 63, 70]))
    it = int(rng.integers(1, 4))
    dt = rng.choice(["u8", "f32", "f64"])
    if dt == "u8": p = rng.integers(0, 256, (b, h, w), dtype=np.uint8)
    elif dt == "f32": p = (rng.random((b, h, w)) * 300 - 50).astype(np.float32)
    else: p = rng.random((b, h, w)) * 1e3 - 200
    got = ctx.iterate(torch.from_numpy(p).cuda(), r, it, mode="exact").cpu().numpy()
    want = np.stack([orc.osbf(c.astype(np.float64), r, it) for c in p])
    ok = np.array_equal(got.view(np.uint64), want.view(np.uint64))
    if not ok:
        bad += 1
        print("MISMATCH", b, h, w, r, it, dt, ctx.last_kernel, int((got != want).sum()))
print(f"fuzz: {n} cases, {bad} mismatches")
