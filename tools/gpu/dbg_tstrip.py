import numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2108_05021_b200 as ob
import oracle
rng = np.random.default_rng(1)
p = rng.random((300, 260)) * 255.0
ctx = ob.Context(0)
got = ctx.iterate(torch.from_numpy(p).cuda(), 2, 2, mode="exact").cpu().numpy()
torch.cuda.synchronize()
want = oracle.Oracle().osbf(p, 2, 2)
print(ctx.last_kernel, "equal:", np.array_equal(got.view(np.uint64), want.view(np.uint64)))
