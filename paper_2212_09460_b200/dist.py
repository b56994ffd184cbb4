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
        # one rank holds the whole accumulator: the peak hint (DESIGN R25) is
        # valid; with several ranks the band partials are summed afterwards
        self.hint_bytes = ld.ld_hough_hint_bytes(1, width, height, n_theta) if world == 1 else 0
        self.hint = (torch.empty((self.hint_bytes,), dtype=torch.uint8, device=self.device)
                     if self.hint_bytes else None)
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
        if self.hint is not None:
            ld.ld_hough_accumulate_hint(self.edges, self.count, self.edge_stride, 1, self.w,
                                        self.h, self.n_theta, self.cos, self.sin, self.acc,
                                        self.hint, self.hint_bytes, stream)
        else:
            ld.ld_hough_accumulate(self.edges, self.count, self.edge_stride, 1, self.w, self.h,
                                   self.n_theta, self.cos, self.sin, self.acc, stream)
        self.launches += ld.ld_last_launch_count()
        allreduce_accumulator(self.acc, self.group)
        if self.hint is not None:
            ld.ld_hough_peaks_hinted(self.acc, 1, self.n_theta, self.n_rho, self.half_theta,
                                     self.half_rho, self.min_votes, self.k, self.hint,
                                     self.hint_bytes, self.peaks, self.n_peaks, self.ws,
                                     self.ws_bytes, stream)
        else:
            ld.ld_hough_peaks(self.acc, 1, self.n_theta, self.n_rho, self.half_theta,
                              self.half_rho, self.min_votes, self.k, self.peaks, self.n_peaks,
                              self.ws, self.ws_bytes, stream)
        self.launches += ld.ld_last_launch_count()
        return self.peaks, self.n_peaks, self.acc, self.count


# ----------------------------------------------------------------------------
# theta-sharded banded detection
# ----------------------------------------------------------------------------
def theta_shard(n_theta: int, rank: int, world: int) -> tuple[int, int]:
    """Theta rows [t0, t1) whose candidates ``rank`` owns (balanced, in order)."""
    return row_band(n_theta, rank, world)


def theta_slice(n_theta: int, half_theta: int, t0: int, t1: int) -> tuple[int, int]:
    """Rows [g0, g1) a shard must vote: its own rows plus every existing row
    within half_theta of them (the peak windows, DESIGN R13)."""
    return max(t0 - half_theta, 0), min(t1 + half_theta, n_theta)


def merge_peak_lists(peaks, n_peaks, n_rho: int, k: int):
    """Merge per-shard top-k lists (global theta bins) into the global top-k.

    peaks: int32 [S][k][3] (theta_bin, rho_bin, votes as uint32 bits), n_peaks
    int32 [S].  Keys are (votes, -theta, -rho) (DESIGN R14) as one int64
    votes * 2^32 + (2^32 - 1 - (theta * n_rho + rho)); runs on the tensors'
    device (no host synchronisation).  Returns (peaks [k][3], n_peaks [1])."""
    import torch
    s, kk, _ = peaks.shape
    p = peaks.reshape(s * kk, 3).to(torch.int64)
    valid = (torch.arange(kk, device=peaks.device)[None, :] < n_peaks[:, None].to(torch.int64))
    valid = valid.reshape(-1)
    votes = p[:, 2] & 0xFFFFFFFF
    idx = p[:, 0] * n_rho + p[:, 1]
    key = votes * (1 << 32) + (0xFFFFFFFF - idx)
    key = torch.where(valid, key, torch.full_like(key, -1))
    top = torch.topk(key, min(k, key.numel())).values
    ok = top >= 0
    idx_out = 0xFFFFFFFF - (top & 0xFFFFFFFF)
    out = torch.full((k, 3), -1, dtype=torch.int64, device=peaks.device)
    out[:, 2] = 0
    n = top.numel()
    out[:n, 0] = torch.where(ok, idx_out // n_rho, torch.full_like(top, -1))
    out[:n, 1] = torch.where(ok, idx_out % n_rho, torch.full_like(top, -1))
    out[:n, 2] = torch.where(ok, top >> 32, torch.zeros_like(top))
    cnt = ok.sum().to(torch.int32).reshape(1)
    return out.to(torch.int32), cnt


class ThetaShardedDetector:
    """Theta-sharded detection of one large image (cfg5, NEXT 1).

    Sobel + binarize + compaction run on this rank's row band (as in
    BandedDetector); the band edge lists are all-gathered (4 B per edge), every
    rank votes ALL edges into only its theta shard plus half_theta halo rows
    (ld_hough_accumulate on a slice of the trig table), finds the candidates of
    its own rows (ld_hough_peaks_ex with global theta bins), and the per-rank
    top-k lists are all-gathered (12 B x k per rank) and merged.  Compared with
    the row-band all_reduce of the 4 n_theta n_rho-byte accumulator this
    exchanges ~4 E bytes, and voting and peaks both scale with the rank count.
    Results are bit-identical to the single-GPU path and the oracle.
    """

    def __init__(self, width, height, n_theta, cos_q15, sin_q15, threshold, k, half_theta,
                 half_rho, min_votes=1, rank=0, world=1, group=None, device=None):
        import torch
        from . import ld
        self.ld = ld
        self.band = BandedDetector(width, height, n_theta, cos_q15, sin_q15, threshold, k,
                                   half_theta, half_rho, min_votes, rank, world, group, device)
        self.device = self.band.device
        self.group, self.rank, self.world = group, rank, world
        self.w, self.h, self.n_theta, self.k = width, height, n_theta, k
        self.half_theta, self.half_rho, self.min_votes = half_theta, half_rho, min_votes
        self.n_rho = self.band.n_rho
        self.t0, self.t1 = theta_shard(n_theta, rank, world)
        self.g0, self.g1 = theta_slice(n_theta, half_theta, self.t0, self.t1)
        c = ld._host_i32(cos_q15)
        s = ld._host_i32(sin_q15)
        self.cos_s, self.sin_s = c[self.g0:self.g1].copy(), s[self.g0:self.g1].copy()
        # gathered edge lists: every rank's band holds at most rows * (W - 2) edges
        self.max_band_edges = max(BandPlan.make(width, height, r, world).max_edges
                                  for r in range(world))
        self.gathered = torch.empty((world, max(self.max_band_edges, 1)), dtype=torch.int32,
                                    device=self.device)
        self.send = torch.zeros((max(self.max_band_edges, 1),), dtype=torch.int32,
                                device=self.device)
        self.all_stride = ld._round_up(max(world * self.max_band_edges, 1), 4)
        self.all_edges = torch.zeros((self.all_stride,), dtype=torch.int32, device=self.device)
        self.total = torch.zeros((1,), dtype=torch.int32, device=self.device)
        ns = max(self.g1 - self.g0, 1)
        self.acc = torch.empty((1, ns, self.n_rho), dtype=torch.int32, device=self.device)
        self.ws_bytes = ld.ld_hough_peaks_workspace_bytes(1, ns, self.n_rho, k)
        self.ws = torch.empty((max(self.ws_bytes, 16),), dtype=torch.uint8, device=self.device)
        self.peaks = torch.empty((1, k, 3), dtype=torch.int32, device=self.device)
        self.n_peaks = torch.empty((1,), dtype=torch.int32, device=self.device)
        self.launches = 0

    def load(self, gray_full):
        self.band.load(gray_full)

    def __call__(self, mark=None):
        """Returns (peaks [1][k][3], n_peaks [1]) on every rank.  `mark(j)`, if
        given, is called at the stage boundaries j = 0 (start), 1 (after
        Sobel), 2 (after the edge exchange), 3 (after voting), 4 (after
        peaks), 5 (after the top-k exchange and merge) -- bench.py records
        CUDA events there."""
        import torch
        import torch.distributed as dist
        ld, b = self.ld, self.band
        mark = mark or (lambda j: None)
        self.launches = 0
        mark(0)
        if b.plan.rows > 0:
            ld.ld_sobel_binarize(b.gray, b.img, b.threshold, None, b.edges, b.edge_stride,
                                 b.count, None)
            self.launches += ld.ld_last_launch_count()
        else:
            b.count.zero_()
        mark(1)
        multi = dist.is_initialized() and self.world > 1
        if multi:
            counts = torch.empty((self.world,), dtype=torch.int32, device=self.device)
            dist.all_gather_into_tensor(counts, b.count, group=self.group)
            cl = counts.tolist()  # host sizes for the variable-length gather
            m = max(max(cl), 1)
            mine = cl[self.rank]
            if mine:
                self.send[:mine].copy_(b.edges[:mine])
            dist.all_gather_into_tensor(self._gbuf(m), self.send[:m], group=self.group)
            parts = [self._gview(m)[r, :cl[r]] for r in range(self.world)]
            n = sum(cl)
            if n:
                torch.cat(parts, out=self.all_edges[:n])
            self.total.fill_(n)
            edges, count, stride = self.all_edges, self.total, self.all_stride
        else:
            edges, count, stride = b.edges, b.count, b.edge_stride
        mark(2)
        self.vote_and_peaks(edges, count, stride, mark)
        if not multi:
            mark(5)
            return self.peaks, self.n_peaks
        allp = torch.empty((self.world, self.k, 3), dtype=torch.int32, device=self.device)
        alln = torch.empty((self.world,), dtype=torch.int32, device=self.device)
        dist.all_gather_into_tensor(allp, self.peaks, group=self.group)
        dist.all_gather_into_tensor(alln, self.n_peaks, group=self.group)
        p, n = merge_peak_lists(allp, alln, self.n_rho, self.k)
        mark(5)
        return p[None], n

    def vote_and_peaks(self, edges, count, stride, mark=None):
        """This rank's theta shard: vote every edge of the image (device list
        `edges`, device `count`) into rows g0 .. g1-1, then the top-k of the
        shard's own rows with global theta bins -> self.peaks, self.n_peaks."""
        ld = self.ld
        if self.g1 > self.g0:
            ld.ld_hough_accumulate(edges, count, stride, 1, self.w, self.h, self.g1 - self.g0,
                                   self.cos_s, self.sin_s, self.acc, None)
            self.launches += ld.ld_last_launch_count()
        if mark:
            mark(3)
        ld.ld_hough_peaks_ex(self.acc, 1, max(self.g1 - self.g0, 1), self.n_rho, self.half_theta,
                             self.half_rho, self.min_votes, self.k, self.t0 - self.g0,
                             self.t1 - self.g0, self.g0, self.peaks, self.n_peaks, self.ws,
                             self.ws_bytes, None)
        self.launches += ld.ld_last_launch_count()
        if mark:
            mark(4)

    def _gbuf(self, m):
        self._gflat = self.gathered.reshape(-1)[: self.world * m]
        return self._gflat

    def _gview(self, m):
        return self._gflat.reshape(self.world, m)
