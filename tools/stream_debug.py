"""Locate fast-mode mismatches against the oracle (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2108_05021_b200 as ob
import oracle

ctx = ob.Context(0)
orc = oracle.Oracle()
for (h, w, r) in [(40, 300, 3), (100, 230, 3), (64, 64, 5), (200, 500, 8)]:
    x = np.random.default_rng(1).random((h, w)) * 255
    got = ctx.iterate(torch.from_numpy(x).cuda(), r, 1, mode="fast").cpu().numpy()
    want = orc.osbf(x, r, 1)
    err = np.abs(got - want)
    bad = np.argwhere(err > 1e-9)
    print(h, w, r, "maxerr", err.max(), "nbad", len(bad))
    if len(bad):
        rows = np.unique(bad[:, 0]); cols = np.unique(bad[:, 1])
        print("  bad rows", rows[:20], "... n", len(rows))
        print("  bad cols", cols[:20], "... n", len(cols))
        y, xx = bad[0]
        print("  first", y, xx, "got", got[y, xx], "want", want[y, xx], "in", x[y, xx])
