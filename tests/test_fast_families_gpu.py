"""Every fast-pass kernel family (selectable with osbf_gpu_set_fast_kernel
for A/B measurements) against the oracle: float input within 1e-5 of the
value range over 3 passes, uint8 first pass bit-exact, band splits equal to
the whole image."""
import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu

FAMILIES = {"arms": range(3, 5), "tma": range(1, 5), "pair": range(1, 5), "tmaseq": range(1, 5), "tmaint": range(1, 5),
            "tile": range(1, 5), "stream": range(5, 17), "strip": range(1, 17), "walk": range(1, 17)}
CASES = [(fam, r) for fam, rs in FAMILIES.items() for r in rs]


@pytest.fixture
def family(request):
    import paper_2108_05021_b200 as ob

    yield
    ob.Context.set_fast_kernel(None)


@pytest.mark.parametrize("fam,r", CASES, ids=[f"{f}-r{r}" for f, r in CASES])
def test_family_matches_oracle(ctx, oracle_lib, family, fam, r):
    import torch

    import paper_2108_05021_b200 as ob

    ob.Context.set_fast_kernel(fam)
    rng = np.random.default_rng(700 + r)
    for shape in [(1, 70, 128), (2, 300, 256), (1, 129, 320), (1, 3, 64)]:
        p = rng.random(shape) * 255.0
        got = ctx.iterate(torch.from_numpy(p).cuda(), r, 3, mode="fast").cpu().numpy()
        assert fam.split("seq")[0] in ctx.last_kernel or fam in ("tile", "tmaseq", "tmaint", "arms"), \
            ctx.last_kernel
        want = np.stack([oracle_lib.osbf(c, r, 3) for c in p])
        assert float(np.abs(got - want).max()) <= 1e-5 * 255.0, shape
    u8 = rng.integers(0, 256, (2, 140, 320), dtype=np.uint8)
    got = ctx.iterate(torch.from_numpy(u8).cuda(), r, 1, mode="fast").cpu().numpy()
    want = np.stack([oracle_lib.osbf(c.astype(np.float64), r, 1) for c in u8])
    assert np.array_equal(bits(got), bits(want))
    f32 = (rng.random((1, 96, 192)) * 8 - 4).astype(np.float32)
    got = ctx.iterate(torch.from_numpy(f32).cuda(), r, 2, mode="fast").cpu().numpy()
    want = oracle_lib.osbf(f32[0].astype(np.float64), r, 2)
    assert float(np.abs(got[0] - want).max()) <= 1e-5 * 8.0
