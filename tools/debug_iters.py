import numpy as np, torch, sys
sys.path.insert(0, '.')
import oracle, paper_2108_05021_b200 as ob
O = oracle.Oracle(); ctx = ob.Context(0)
rng = np.random.default_rng(0)
for (h, w, dt) in [(64, 64, np.float64), (256, 256, np.float32), (128, 128, np.float32), (33, 45, np.float32)]:
    x = (rng.random((h, w)) * 255).astype(dt)
    for it in (1, 2, 3, 4):
        want = O.osbf(x, 2, it)
        for mode in ("exact", "fast"):
            t = torch.from_numpy(x).cuda()
            got = ctx.iterate(t, 2, it, mode=mode)
            torch.cuda.synchronize()
            g = got.cpu().numpy()
            print(h, w, dt.__name__, it, mode, 'maxdiff', float(np.abs(g - want).max()), 'zeros', int((g == 0).sum()), 'err', ctx._lib.osbf_gpu_last_error())
