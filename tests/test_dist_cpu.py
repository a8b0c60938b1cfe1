"""Multi-rank host logic on CPU (world_size 2, gloo): batch sharding and the
row-band partition with per-pass halo exchange.  The per-band compute here is
the CPU oracle applied to the halo'd band buffer (test stand-in for the GPU
kernel's step_band); the exchange, offsets and border handling are the code
under test."""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_batch_covers_everything():
    from paper_2108_05021_b200.dist import shard_batch

    for batch in (1, 7, 256):
        for world in (1, 2, 3, 8):
            seen = []
            for rank in range(world):
                s, n = shard_batch(batch, world, rank)
                seen.extend(range(s, s + n))
            assert seen == list(range(batch))


def test_band_rows_alignment_and_limits():
    from paper_2108_05021_b200.dist import band_rows

    bands = band_rows(32768, 8, 4)
    assert bands[0][0] == 0 and bands[-1][1] == 32768
    assert all(r0 % 64 == 0 for r0, _ in bands)
    assert all(b[1] == nb[0] for b, nb in zip(bands, bands[1:]))
    with pytest.raises(ValueError):
        band_rows(10, 8, 4)


def _oracle_band_step(src, lay, dst_band):
    """CPU stand-in for step_band: the oracle on the halo'd buffer.  Windows of
    band rows reach at most r rows past the band, i.e. inside the halos, and
    the buffer ends exactly where the image does."""
    import torch

    import oracle

    out = oracle.Oracle().osbf_step(src.numpy(), lay.radius)
    dst_band.copy_(torch.from_numpy(out[lay.halo_top:lay.halo_top + lay.rows]))


def _worker(rank, world, port, h, w, r, iters, seed, result_path):
    import torch
    import torch.distributed as dist

    from paper_2108_05021_b200.dist import BandLayout, RowBandOSBF

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    img = np.random.default_rng(seed).random((h, w)) * 255.0
    lay = BandLayout.make(h, w, r, world, rank)
    band = torch.from_numpy(img[lay.row0:lay.row1].copy())
    out = RowBandOSBF(lay, rank, world, step=_oracle_band_step).run(band, iters)
    if rank == 0:
        parts = [out]
        for k in range(1, world):
            part = torch.zeros((BandLayout.make(h, w, r, world, k).rows, w), dtype=torch.float64)
            dist.recv(part, src=k)
            parts.append(part)
        np.save(result_path, torch.cat(parts).numpy())
    else:
        dist.send(out.contiguous(), dst=0)
    dist.destroy_process_group()


@pytest.mark.parametrize("h,w,r,iters", [(300, 40, 2, 3), (256, 33, 5, 2), (130, 20, 16, 2)])
def test_row_bands_over_gloo_match_whole_image(tmp_path, h, w, r, iters):
    import torch.multiprocessing as mp

    import oracle

    world = 2
    path = str(tmp_path / "out.npy")
    mp.start_processes(_worker, args=(world, _free_port(), h, w, r, iters, 7, path), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(path)
    img = np.random.default_rng(7).random((h, w)) * 255.0
    want = oracle.Oracle().osbf(img, r, iters)
    # bands re-base the prefix sums (like the fast mode); selection may flip
    # only on sub-ulp near-ties, so compare with the float tolerance
    assert got.shape == want.shape
    assert np.abs(got - want).max() <= 1e-5 * 255.0


def test_row_bands_integer_first_pass_bit_exact(tmp_path):
    """Integer-valued input: every window sum is exact in any order, so the
    banded first pass is bit-identical to the whole image."""
    import torch.multiprocessing as mp

    import oracle

    h, w, r = 200, 31, 3
    path = str(tmp_path / "out.npy")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    mp.start_processes(_worker_int, args=(2, _free_port(), h, w, r, path), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(path)
    img = np.random.default_rng(3).integers(0, 256, (h, w)).astype(np.float64)
    want = oracle.Oracle().osbf(img, r, 1)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def _worker_int(rank, world, port, h, w, r, path):
    import torch
    import torch.distributed as dist

    from paper_2108_05021_b200.dist import BandLayout, RowBandOSBF

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    img = np.random.default_rng(3).integers(0, 256, (h, w)).astype(np.float64)
    lay = BandLayout.make(h, w, r, world, rank)
    out = RowBandOSBF(lay, rank, world, step=_oracle_band_step).run(
        torch.from_numpy(img[lay.row0:lay.row1].copy()), 1)
    if rank == 0:
        other = torch.zeros((BandLayout.make(h, w, r, world, 1).rows, w), dtype=torch.float64)
        dist.recv(other, src=1)
        np.save(path, torch.cat([out, other]).numpy())
    else:
        dist.send(out.contiguous(), dst=0)
    dist.destroy_process_group()
