"""Multi-GPU OSBF: one process per GPU, torch.distributed for the plumbing.

Two partitionings:

* **Batch sharding** (:func:`shard_batch`) — independent planes (C4's 256
  images, colour channels) split across ranks; no data-path collective.
* **Row bands** (:class:`RowBandOSBF`) — one image too large or too slow for
  one GPU (C5, 32768²) split into horizontal bands.  Each pass needs the
  ``r`` rows just outside the band, so after every pass each rank sends its
  first/last ``r`` rows to its neighbours (NCCL send/recv over NVLink on the
  GPU; any backend works — the CPU tests run it over gloo).  Every band's
  pass is one ``osbf_gpu_step_band`` launch that clips windows at the GLOBAL
  image border, so the bands together compute exactly the whole-image fast
  pass (bit-identical when band starts are multiples of the 64-row tile,
  which :func:`band_rows` arranges).

Only the fast mode partitions: the exact mode replays the reference's
whole-image serial prefix (integral.hpp:20-29), a dependency chain over the
full height — it shards by batch only.
"""
from __future__ import annotations

from dataclasses import dataclass

TILE_ROWS = 64  # fast-kernel tile height; band starts aligned to it


def shard_batch(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, start+count) share of a batch for ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def band_rows(height: int, world: int, radius: int, align: int = TILE_ROWS) -> list[tuple[int, int]]:
    """Split ``height`` rows into ``world`` bands [row0, row1), starts aligned
    to ``align`` where possible; every band has at least ``radius`` rows so a
    neighbour's halo lies in one band."""
    if world < 1:
        raise ValueError("world must be >= 1")
    bounds = [0]
    for i in range(1, world):
        b = round(height * i / world / align) * align
        if b <= bounds[-1]:
            b = bounds[-1] + max(1, height // world)
        bounds.append(min(b, height))
    bounds.append(height)
    bands = list(zip(bounds[:-1], bounds[1:]))
    for r0, r1 in bands:
        if r1 - r0 < max(1, radius):
            raise ValueError(f"band [{r0},{r1}) shorter than the radius {radius}: too many ranks")
    return bands


@dataclass(frozen=True)
class BandLayout:
    """Where one rank's band sits: buffer rows = [halo_top | band | halo_bot]."""

    height: int
    width: int
    radius: int
    row0: int
    row1: int
    halo_top: int
    halo_bot: int

    @property
    def rows(self) -> int:
        return self.row1 - self.row0

    @property
    def buf_rows(self) -> int:
        return self.halo_top + self.rows + self.halo_bot

    @property
    def buf_row0(self) -> int:  # global row of buffer row 0
        return self.row0 - self.halo_top

    @staticmethod
    def make(height: int, width: int, radius: int, world: int, rank: int) -> "BandLayout":
        r0, r1 = band_rows(height, world, radius)[rank]
        return BandLayout(height, width, radius, r0, r1, min(radius, r0),
                          min(radius, height - r1))


def exchange_halos(buf, lay: BandLayout, rank: int, world: int, group=None) -> None:
    """Fill buf's halo rows from the neighbours' band rows (both directions),
    with batched point-to-point send/recv (NCCL or gloo)."""
    import torch.distributed as dist

    ops = []
    top = lay.halo_top
    band = buf[top:top + lay.rows]
    if rank > 0 and lay.halo_top:
        ops.append(dist.P2POp(dist.isend, band[:lay.halo_top].contiguous(), rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, buf[:top], rank - 1, group))
    if rank < world - 1 and lay.halo_bot:
        ops.append(dist.P2POp(dist.isend, band[lay.rows - lay.halo_bot:].contiguous(), rank + 1,
                              group))
        ops.append(dist.P2POp(dist.irecv, buf[top + lay.rows:], rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


class RowBandOSBF:
    """Iterate the fast OSBF over this rank's row band with per-pass halo
    exchange.  ``step(src_buf, lay, dst_band)`` computes one pass of the band
    rows from the halo'd buffer; by default it is the GPU kernel
    (``Context.step_band``)."""

    def __init__(self, lay: BandLayout, rank: int, world: int, step=None, group=None,
                 device=None):
        self.lay, self.rank, self.world, self.group = lay, rank, world, group
        self.device = device
        self.step = step or self._gpu_step
        self._ctx = None

    def _gpu_step(self, src, lay: BandLayout, dst_band) -> None:
        if self._ctx is None:
            from .api import Context

            self._ctx = Context(src.device.index or 0)
        self._ctx.step_band(src, lay.buf_row0, dst_band, lay.row0, lay.rows, lay.height,
                            lay.radius, mode="fast")

    def buffers(self, device):
        """The two halo'd fp64 ping-pong buffers (allocated once, reused)."""
        import torch

        lay = self.lay
        if getattr(self, "_bufs", None) is None or self._bufs[0].device != device:
            self._bufs = [torch.zeros((lay.buf_rows, lay.width), dtype=torch.float64,
                                      device=device) for _ in range(2)]
        return self._bufs

    def run(self, band, iterations: int):
        """``band``: this rank's rows [row0, row1) (any float dtype, on the
        compute device); returns the filtered band (a float64 view into the
        rank's buffers, valid until the next run)."""
        lay = self.lay
        if tuple(band.shape) != (lay.rows, lay.width):
            raise ValueError(f"band shape {tuple(band.shape)} != {(lay.rows, lay.width)}")
        bufs = self.buffers(band.device)
        top = lay.halo_top
        bufs[0][top:top + lay.rows].copy_(band)
        if iterations == 0:
            return bufs[0][top:top + lay.rows]
        exchange_halos(bufs[0], lay, self.rank, self.world, self.group)
        cur = 0
        for it in range(iterations):
            src, dst = bufs[cur], bufs[1 - cur]
            self.step(src, lay, dst[top:top + lay.rows])
            if it + 1 < iterations:
                exchange_halos(dst, lay, self.rank, self.world, self.group)
            cur = 1 - cur
        return bufs[cur][top:top + lay.rows]
