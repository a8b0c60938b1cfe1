"""Multi-GPU OSBF: one process per GPU, torch.distributed for the plumbing.

Two partitionings:

* **Batch sharding** (:func:`shard_batch`) — independent planes (C4's 256
  images, colour channels) split across ranks; no data-path collective.
* **Row bands** (:class:`RowBandOSBF`) — one image too large or too slow for
  one GPU (C5, 32768²) split into horizontal bands.  Each pass needs the
  ``r`` rows just outside the band.  Two exchanges: ``nccl`` (after every
  pass each rank sends its first/last ``r`` rows to its neighbours, batched
  send/recv; any backend works — the CPU tests run it over gloo) and
  ``push`` (the pass kernel itself stores those rows into the neighbours'
  halo rows in symmetric memory, then a device-side barrier).  Every band's
  pass is one launch that clips windows at the GLOBAL image border, so the
  bands together compute the whole-image fast pass (bit-identical for the
  tile kernels when band starts are multiples of the 64-row tile, which
  :func:`band_rows` arranges; within fp64 rounding for the streaming r=5..7
  kernel).

Only the fast mode partitions: the exact mode replays the reference's
whole-image serial prefix (integral.hpp:20-29), a dependency chain over the
full height — it shards by batch only.
"""
from __future__ import annotations

from dataclasses import dataclass

TILE_ROWS = 128  # fast tile-kernel height (r <= 2); band starts aligned to it
WALK_ROWS = 512  # fast column-walk row block (r >= 3): preferred band alignment


def shard_batch(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, start+count) share of a batch for ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def _split(height: int, world: int, align: int) -> list[tuple[int, int]]:
    bounds = [0]
    for i in range(1, world):
        b = round(height * i / world / align) * align
        if b <= bounds[-1]:
            b = bounds[-1] + max(1, height // world)
        bounds.append(min(b, height))
    bounds.append(height)
    return list(zip(bounds[:-1], bounds[1:]))


def band_rows(height: int, world: int, radius: int, align: int | None = None) -> list[tuple[int, int]]:
    """Split ``height`` rows into ``world`` bands [row0, row1), starts aligned
    to ``align`` where possible (default: the column walk's 512-row block when
    every band can hold one, else the 128-row tile; aligned bands give results
    bit-identical to the whole image).  Every band has at least ``radius``
    rows so a neighbour's halo lies in one band; when an aligned split cannot
    give that, the split falls back to a coarser-then-unaligned one."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if align is not None:
        aligns = [align]
    elif height >= world * WALK_ROWS:
        aligns = [WALK_ROWS, TILE_ROWS]
    else:
        aligns = [TILE_ROWS]
    for a in aligns + [1]:
        bands = _split(height, world, a)
        if all(r1 - r0 >= max(1, radius) for r0, r1 in bands):
            return bands
    raise ValueError(f"{height} rows cannot give {world} bands of at least the radius {radius}: "
                     "too many ranks")


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
    """Iterate the fast OSBF over this rank's row band.

    ``exchange="nccl"``: after every pass the boundary rows go to the
    neighbours with batched send/recv (:func:`exchange_halos`).

    ``exchange="push"``: the exchange is fused into the pass
    (``osbf_gpu_step_band_push``): the kernel that computes the band also
    stores its first / last ``r`` output rows straight into the neighbours'
    halo rows, which live in symmetric memory (``torch.distributed.
    _symmetric_memory``: peer-mapped over NVLink), and a device-side barrier
    orders the next pass.  No separate copy or collective touches the halos.

    ``step(src_buf, lay, dst_band, push)`` computes one pass (default: the GPU
    kernel).  ``peer_buffers`` / ``sync`` override the symmetric-memory
    plumbing (tests emulate several ranks on one device with them)."""

    def __init__(self, lay: BandLayout, rank: int, world: int, step=None, group=None,
                 device=None, exchange: str = "nccl", peer_buffers=None, sync=None):
        if exchange not in ("nccl", "push"):
            raise ValueError("exchange must be 'nccl' or 'push'")
        self.lay, self.rank, self.world, self.group = lay, rank, world, group
        self.device = device
        self.exchange = exchange
        self.step = step or self._gpu_step
        self._ctx = None
        self._peer_buffers = peer_buffers
        self._sync = sync
        self._bufs = None
        self.exchange_note = None

    def _gpu_step(self, src, lay: BandLayout, dst_band, push=None) -> None:
        if self._ctx is None:
            from .api import Context

            self._ctx = Context(src.device.index or 0)
        up, down = push if push else (None, None)
        self._ctx.step_band(src, lay.buf_row0, dst_band, lay.row0, lay.rows, lay.height,
                            lay.radius, mode="fast", push_up=up, push_down=down,
                            push_rows=lay.radius if push else 0)

    # -- buffers -----------------------------------------------------------
    def _layouts(self):
        lay = self.lay
        return [BandLayout.make(lay.height, lay.width, lay.radius, self.world, q)
                for q in range(self.world)]

    def buffers(self, device):
        """The two halo'd fp64 ping-pong buffers (allocated once, reused).
        Push mode: both live in one symmetric allocation of the same size on
        every rank (the largest band's), so a neighbour can address them."""
        import torch

        lay = self.lay
        if self._bufs is not None and self._bufs[0].device == device:
            return self._bufs
        if self.exchange == "nccl" or (self.world == 1 and self._peer_buffers is None):
            self._bufs = [torch.zeros((lay.buf_rows, lay.width), dtype=torch.float64,
                                      device=device) for _ in range(2)]
            return self._bufs
        self._slot = max(q.buf_rows for q in self._layouts()) * lay.width
        if self._peer_buffers is None:
            import torch.distributed as dist

            try:
                import torch.distributed._symmetric_memory as symm_mem

                flat = symm_mem.empty(2 * self._slot, dtype=torch.float64, device=device)
                hdl = symm_mem.rendezvous(flat, self.group or dist.group.WORLD)
            except Exception as e:  # no peer-mappable memory on this system
                # the exchange mechanism (not the filter) falls back to NCCL
                # send/recv, recorded in exchange_note; every rank takes the
                # same branch because rendezvous is collective
                self.exchange = "nccl"
                self.exchange_note = f"symmetric memory unavailable ({type(e).__name__}: {e})"
                return self.buffers(device)
            self._hdl = hdl
            self._flat = flat
            self._peer_buffers = lambda q: hdl.get_buffer(q, (2 * self._slot,), torch.float64)
            if self._sync is None:
                self._sync = lambda: hdl.barrier(channel=0)
        flat = self._peer_buffers(self.rank)
        flat.zero_()
        self._bufs = [flat[k * self._slot:k * self._slot + lay.buf_rows * lay.width]
                      .view(lay.buf_rows, lay.width) for k in range(2)]
        return self._bufs

    def _push_targets(self, k: int):
        """Views of the neighbours' halo rows in their buffer ``k``: the upper
        neighbour's bottom halo (= this band's first r rows) and the lower
        neighbour's top halo (= this band's last r rows)."""
        lays, lay, w = self._layouts(), self.lay, self.lay.width
        up = down = None
        if self.rank > 0 and lay.halo_top:
            q = lays[self.rank - 1]
            flat = self._peer_buffers(self.rank - 1)
            off = k * self._slot + (q.halo_top + q.rows) * w
            up = flat[off:off + q.halo_bot * w].view(q.halo_bot, w)
        if self.rank < self.world - 1 and lay.halo_bot:
            flat = self._peer_buffers(self.rank + 1)
            off = k * self._slot
            down = flat[off:off + lays[self.rank + 1].halo_top * w].view(-1, w)
        return up, down

    # -- passes ------------------------------------------------------------
    def prime(self, band):
        """Load this rank's rows [row0, row1) and exchange the initial halos."""
        lay = self.lay
        if tuple(band.shape) != (lay.rows, lay.width):
            raise ValueError(f"band shape {tuple(band.shape)} != {(lay.rows, lay.width)}")
        bufs = self.buffers(band.device)
        top = lay.halo_top
        bufs[0][top:top + lay.rows].copy_(band)
        self._cur = 0

    def exchange_initial(self):
        if self.world > 1:
            exchange_halos(self._bufs[0], self.lay, self.rank, self.world, self.group)

    def one_pass(self, last: bool):
        """One pass from buffer cur into buffer 1 - cur, halos included."""
        lay, bufs, top = self.lay, self._bufs, self.lay.halo_top
        src, dst = bufs[self._cur], bufs[1 - self._cur]
        if self.exchange == "push" and self.world > 1:
            self.step(src, lay, dst[top:top + lay.rows], self._push_targets(1 - self._cur))
        else:
            self.step(src, lay, dst[top:top + lay.rows])
            if not last and self.world > 1:
                exchange_halos(dst, lay, self.rank, self.world, self.group)
        self._cur = 1 - self._cur

    def result(self):
        top = self.lay.halo_top
        return self._bufs[self._cur][top:top + self.lay.rows]

    def run(self, band, iterations: int):
        """``band``: this rank's rows [row0, row1) (any float dtype, on the
        compute device); returns the filtered band (a float64 view into the
        rank's buffers, valid until the next run)."""
        self.prime(band)
        if iterations == 0:
            return self.result()
        if self.exchange == "push" and self.world > 1:
            self._sync()  # neighbours done with the previous run's pushes
        self.exchange_initial()
        for it in range(iterations):
            self.one_pass(last=it + 1 == iterations)
            if self.exchange == "push" and self.world > 1:
                self._sync()  # every push landed before anyone reads its halos
        return self.result()
