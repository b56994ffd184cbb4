"""Multi-GPU partitioning of the hot path.

One process per GPU, ``torch.distributed`` for the plumbing.  Two partitions:

* **frame shards** (cfg3, cfg4): a batch of independent frames splits into
  contiguous per-rank ranges; every rank runs the whole path on its frames with
  no data-path collective (weak scaling).
* **row bands** (cfg5): one large image splits into bands of rows.  Each rank
  runs the fused Sobel + binarize + compaction on its band (1-row halo, global
  border semantics via ``ld_image.row_begin/row_end``), votes its global-y
  edges into a full-size partial accumulator, and the partial accumulators are
  summed with one ``all_reduce(SUM)`` -- the only exchange step of the method
  (the Hough transform is additive over edge sets, SURVEY §8(c) pins).  Peaks
  then run on every rank and are identical.

The accumulator is ``uint32`` (DESIGN R12) held in an ``int32`` tensor; the SUM
is exact because every count is at most W*H < 2^31.  All arithmetic of the
method stays in libld.so; this module only partitions, moves and reduces.
"""
from __future__ import annotations

from dataclasses import dataclass


def frame_shard(n_frames: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced shard of ``n_frames``: (first, count) of ``rank``."""
    if world < 1 or not 0 <= rank < world or n_frames < 0:
        raise ValueError("bad shard request")
    base, extra = divmod(n_frames, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def row_band(height: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [row_begin, row_end) owned by ``rank``: balanced, contiguous, in
    rank order; empty (row_begin == row_end) when height < world."""
    first, count = frame_shard(height, rank, world)
    return first, first + count


def band_read_rows(height: int, row_begin: int, row_end: int) -> tuple[int, int]:
    """Input rows a band must read: its own rows plus a 1-row halo on each side
    (clipped to the image), as ld.h's ld_image contract requires."""
    return max(row_begin - 1, 0), min(row_end + 1, height)


def allreduce_accumulator(acc, group=None):
    """Sum the ranks' partial accumulators in place (uint32 bits in an int32
    tensor; exact, see the module docstring).  NCCL on GPU tensors, gloo on
    CPU tensors."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    return acc


@dataclass
class BandPlan:
    width: int
    height: int
    rank: int
    world: int
    row_begin: int
    row_end: int
    read_begin: int
    read_end: int

    @classmethod
    def make(cls, width: int, height: int, rank: int, world: int) -> "BandPlan":
        rb, re = row_band(height, rank, world)
        r0, r1 = band_read_rows(height, rb, re)
        return cls(width, height, rank, world, rb, re, r0, r1)

    @property
    def rows(self) -> int:
        return self.row_end - self.row_begin

    @property
    def max_edges(self) -> int:
        return self.rows * max(self.width - 2, 0)


class BandedDetector:
    """Row-band detector of one large image on this rank (cfg5).

    ``load(gray)`` copies this rank's band (with halo) of a full uint8 [H][W]
    image to the device once; ``__call__`` then runs, on ``stream``:
    ld_sobel_binarize(band) -> ld_hough_accumulate(full-size partial acc) ->
    all_reduce(SUM) -> ld_hough_peaks, and returns (peaks, n_peaks, acc, count).
    """

    def __init__(self, width, height, n_theta, cos_q15, sin_q15, threshold, k, half_theta,
                 half_rho, min_votes=1, rank=0, world=1, group=None, device=None):
        import torch
        from . import ld
        self.ld = ld
        self.plan = BandPlan.make(width, height, rank, world)
        self.device = torch.device("cuda") if device is None else device
        self.group = group
        self.w, self.h, self.n_theta = width, height, n_theta
        self.cos, self.sin = ld._host_i32(cos_q15), ld._host_i32(sin_q15)
        self.threshold, self.k = threshold, k
        self.half_theta, self.half_rho, self.min_votes = half_theta, half_rho, min_votes
        self.pitch = ld._round_up(width, 16)
        self.n_rho = 2 * ld.ld_rho_offset(width, height) + 1
        p = self.plan
        self.img = (ld.make_image(width, height, self.pitch, (p.read_end - p.read_begin) * self.pitch,
                                  1, p.row_begin, p.row_end) if p.rows > 0 else None)
        self.gray = torch.zeros((max(p.read_end - p.read_begin, 1), self.pitch), dtype=torch.uint8,
                                device=self.device)
        self.edge_stride = ld._round_up(max(p.max_edges, 1), 4)
        self.edges = torch.empty((self.edge_stride,), dtype=torch.int32, device=self.device)
        self.count = torch.zeros((1,), dtype=torch.int32, device=self.device)
        self.acc = torch.empty((1, n_theta, self.n_rho), dtype=torch.int32, device=self.device)
        self.ws_bytes = ld.ld_hough_peaks_workspace_bytes(1, n_theta, self.n_rho, k)
        self.ws = torch.empty((max(self.ws_bytes, 16),), dtype=torch.uint8, device=self.device)
        self.peaks = torch.empty((1, k, 3), dtype=torch.int32, device=self.device)
        self.n_peaks = torch.empty((1,), dtype=torch.int32, device=self.device)
        self.launches = 0

    def load(self, gray_full):
        """gray_full: uint8 [H][W] (numpy or torch, host or device)."""
        import torch
        p = self.plan
        if p.rows == 0:
            return
        band = gray_full[p.read_begin:p.read_end]
        if not isinstance(band, torch.Tensor):
            band = torch.from_numpy(band.copy())
        self.gray[:, :self.w].copy_(band)

    def __call__(self, stream=None):
        import torch
        if stream is not None and not isinstance(stream, int):
            with torch.cuda.stream(stream):  # the collective orders on torch's current stream
                return self._run(None)
        return self._run(stream)

    def _run(self, stream):
        ld = self.ld
        self.launches = 0
        if self.plan.rows > 0:
            ld.ld_sobel_binarize(self.gray, self.img, self.threshold, None, self.edges,
                                 self.edge_stride, self.count, stream)
            self.launches += ld.ld_last_launch_count()
        else:
            self.count.zero_()
        ld.ld_hough_accumulate(self.edges, self.count, self.edge_stride, 1, self.w, self.h,
                               self.n_theta, self.cos, self.sin, self.acc, stream)
        self.launches += ld.ld_last_launch_count()
        allreduce_accumulator(self.acc, self.group)
        ld.ld_hough_peaks(self.acc, 1, self.n_theta, self.n_rho, self.half_theta, self.half_rho,
                          self.min_votes, self.k, self.peaks, self.n_peaks, self.ws, self.ws_bytes,
                          stream)
        self.launches += ld.ld_last_launch_count()
        return self.peaks, self.n_peaks, self.acc, self.count
