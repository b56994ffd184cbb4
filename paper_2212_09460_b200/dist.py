"""Multi-GPU partitioning of the hot path.

One process per GPU, ``torch.distributed`` for the plumbing.  Two partitions:

* **frame shards** (cfg3, cfg4): a batch of independent frames splits into
  contiguous per-rank ranges (BASELINE.json: the batch "sharded across
  1/2/4/8 GPUs", i.e. strong scaling of a fixed batch; bench.py --scaling weak
  gives every rank a whole batch instead); every rank runs the whole path on
  its frames with no data-path collective.
* **row bands** (cfg5): one large image splits into bands of rows.  Each rank
  runs the fused Sobel + binarize + compaction on its band (1-row halo, global
  border semantics via ``ld_image.row_begin/row_end``), votes its global-y
  edges into a full-size partial accumulator, and the partial accumulators are
  summed with one ``all_reduce(SUM)`` -- the only exchange step of the method
  (the Hough transform is additive over edge sets, SURVEY §8(c) pins).  Peaks
  then run on every rank and are identical.
* **theta shards** (cfg5, NEXT 1): row bands for Sobel, the band edge sets
  exchanged as fixed-size bitmaps (all_gather, no host synchronisation), each
  rank votes all edges into its own theta rows (+ halo) and the per-rank top-k
  lists are all-gathered and merged on the device.

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
    image to the device once; ``__call__`` then runs, on the current stream
    (or ``stream``): ld_sobel_binarize(band) -> ld_hough_accumulate(full-size
    partial acc) -> all_reduce(SUM) -> ld_hough_peaks, and returns (peaks,
    n_peaks, acc, count).  ``mark(j)``, if given, is called at the stage
    boundaries j = 0 (start), 1 (after Sobel), 2 (after voting), 3 (after the
    all_reduce), 4 (after peaks) -- bench.py records CUDA events there.
    """

    def __init__(self, width, height, n_theta, cos_q15, sin_q15, threshold, k, half_theta,
                 half_rho, min_votes=1, rank=0, world=1, group=None, device=None):
        import torch
        from . import ld
        self.ld = ld
        self.plan = BandPlan.make(width, height, rank, world)
        self.device = torch.device("cuda") if device is None else device
        self.group, self.world = group, world
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
        # peak hint (DESIGN R25, R30): one rank holds the whole accumulator, so
        # voting records it; with several ranks the band partials are summed
        # afterwards and the hint is taken from the sum (ld_hough_hint_from_acc)
        self.hint_bytes = ld.ld_hough_hint_bytes(1, width, height, n_theta)
        self.hint = torch.empty((self.hint_bytes,), dtype=torch.uint8, device=self.device)
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

    @property
    def result(self):
        return self.peaks, self.n_peaks

    def __call__(self, stream=None, mark=None):
        import torch
        if isinstance(stream, int):  # a raw cudaStream_t handle
            stream = torch.cuda.ExternalStream(stream, device=self.device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        # one stream for the kernels AND the collective (NCCL orders on torch's
        # current stream), so the all_reduce sums finished partials
        with torch.cuda.device(self.device), torch.cuda.stream(stream):
            return self._run(stream, mark or (lambda j: None))

    def _run(self, stream, mark):
        ld = self.ld
        self.launches = 0
        mark(0)
        if self.plan.rows > 0:
            ld.ld_sobel_binarize(self.gray, self.img, self.threshold, None, self.edges,
                                 self.edge_stride, self.count, stream)
            self.launches += ld.ld_last_launch_count()
        else:
            self.count.zero_()
        mark(1)
        whole = self.world == 1
        ld.ld_hough_accumulate_opt(self.edges, self.count, self.edge_stride, 1, self.w, self.h,
                                   self.n_theta, self.cos, self.sin, 0, self.acc,
                                   self.hint if whole else None,
                                   self.hint_bytes if whole else 0, stream)
        self.launches += ld.ld_last_launch_count()
        mark(2)
        allreduce_accumulator(self.acc, self.group)
        mark(3)
        if not whole:
            ld.ld_hough_hint_from_acc(self.acc, 1, self.n_theta, self.n_rho, 0, self.n_theta,
                                      self.hint, self.hint_bytes, stream)
            self.launches += ld.ld_last_launch_count()
        ld.ld_hough_peaks_opt(self.acc, 1, self.n_theta, self.n_rho, self.half_theta,
                              self.half_rho, self.min_votes, self.k, 0, self.n_theta, 0,
                              self.hint, self.hint_bytes, 0, self.peaks, self.n_peaks, self.ws,
                              self.ws_bytes, stream)
        self.launches += ld.ld_last_launch_count()
        mark(4)
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


def merge_peak_lists(peaks, n_peaks, n_rho: int, k: int, stream=None):
    """Merge per-shard top-k lists (global theta bins) into the global top-k
    on the device (libld ld_merge_peak_lists, key (votes, -theta, -rho), DESIGN
    R14; no host synchronisation).  peaks: int32 [S][k][3], n_peaks int32 [S].
    Returns (peaks [k][3], n_peaks [1])."""
    import torch
    from . import ld
    s = peaks.shape[0]
    out = torch.empty((k, 3), dtype=torch.int32, device=peaks.device)
    n = torch.empty((1,), dtype=torch.int32, device=peaks.device)
    ld.ld_merge_peak_lists(peaks.contiguous(), n_peaks.contiguous(), s, k, n_rho, out, n, stream)
    return out, n


class ThetaShardedDetector:
    """Theta-sharded detection of one large image (cfg5, NEXT 1).

    Sobel + binarize + compaction run on this rank's row band (as in
    BandedDetector); the band's edge set is turned into a fixed-size bitmap
    (ld_edges_to_bitmask, 1 bit per band pixel) and the bitmaps are
    all-gathered -- fixed-size, so no host-known sizes and no host
    synchronisation -- and expanded back into one edge list of the whole image
    on every rank (ld_bitmask_to_edges).  Every rank then votes ALL edges into
    only its theta shard plus half_theta halo rows (ld_hough_accumulate on a
    slice of the trig table), finds the candidates of its own rows
    (ld_hough_peaks_ex with global theta bins), and the per-rank top-k lists
    are all-gathered (12 B x k per rank) and merged on the device
    (ld_merge_peak_lists).  Compared with the row-band all_reduce of the
    4 n_theta n_rho-byte accumulator (47.5 MB for cfg5) this exchanges W*H/8
    bytes (2.1 MB), and voting and peaks both scale with the rank count.
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
        # band bitmaps: every rank's block has the largest band's row count
        plans = [BandPlan.make(width, height, r, world) for r in range(world)]
        self.block_rows = [p.rows for p in plans]
        self.block_begin = [p.row_begin for p in plans]
        self.stride_rows = max(max(self.block_rows), 1)
        self.words = ld.ld_edge_bitmask_words(width, self.stride_rows)
        self.bits = torch.zeros((self.words,), dtype=torch.int32, device=self.device)
        self.all_bits = torch.zeros((world * self.words,), dtype=torch.int32, device=self.device)
        self.all_stride = ld._round_up(max(height * width, 1), 4)
        self.all_edges = torch.zeros((self.all_stride,), dtype=torch.int32, device=self.device)
        self.total = torch.zeros((1,), dtype=torch.int32, device=self.device)
        ns = max(self.g1 - self.g0, 1)
        self.acc = torch.empty((1, ns, self.n_rho), dtype=torch.int32, device=self.device)
        self.ws_bytes = ld.ld_hough_peaks_workspace_bytes(1, ns, self.n_rho, k)
        self.ws = torch.empty((max(self.ws_bytes, 16),), dtype=torch.uint8, device=self.device)
        self.hint_bytes = ld.ld_hough_hint_bytes(1, width, height, ns)
        self.hint = torch.empty((self.hint_bytes,), dtype=torch.uint8, device=self.device)
        self.peaks = torch.empty((1, k, 3), dtype=torch.int32, device=self.device)
        self.n_peaks = torch.empty((1,), dtype=torch.int32, device=self.device)
        self.allp = torch.empty((world, k, 3), dtype=torch.int32, device=self.device)
        self.alln = torch.empty((world,), dtype=torch.int32, device=self.device)
        self.out_peaks = torch.empty((k, 3), dtype=torch.int32, device=self.device)
        self.out_n = torch.empty((1,), dtype=torch.int32, device=self.device)
        self.launches = 0

    def load(self, gray_full):
        self.band.load(gray_full)

    @property
    def result(self):
        """(peaks [k][3], n_peaks [1]) of the last call, identical on every rank."""
        return self.out_peaks, self.out_n

    def __call__(self, mark=None):
        """Returns (peaks [k][3], n_peaks [1]) on every rank, on the current
        stream.  `mark(j)`, if given, is called at the stage boundaries j = 0
        (start), 1 (after Sobel), 2 (after the edge exchange), 3 (after
        voting), 4 (after peaks), 5 (after the top-k exchange and merge) --
        bench.py records CUDA events there."""
        import torch
        import torch.distributed as dist
        ld, b = self.ld, self.band
        mark = mark or (lambda j: None)
        self.launches = 0
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device)
            mark(0)
            if b.plan.rows > 0:
                ld.ld_sobel_binarize(b.gray, b.img, b.threshold, None, b.edges, b.edge_stride,
                                     b.count, stream)
                self.launches += ld.ld_last_launch_count()
            else:
                b.count.zero_()
            mark(1)
            multi = dist.is_initialized() and self.world > 1
            if multi:
                ld.ld_edges_to_bitmask(b.edges, b.count, self.w, b.plan.row_begin,
                                       self.stride_rows, self.bits, stream)
                self.launches += ld.ld_last_launch_count()
                dist.all_gather_into_tensor(self.all_bits, self.bits, group=self.group)
                ld.ld_bitmask_to_edges(self.all_bits, self.w, self.block_begin, self.block_rows,
                                       self.stride_rows, self.all_edges, self.all_stride,
                                       self.total, stream)
                self.launches += ld.ld_last_launch_count()
                edges, count, stride = self.all_edges, self.total, self.all_stride
            else:
                edges, count, stride = b.edges, b.count, b.edge_stride
            mark(2)
            self.vote_and_peaks(edges, count, stride, mark)
            if multi:
                dist.all_gather_into_tensor(self.allp, self.peaks, group=self.group)
                dist.all_gather_into_tensor(self.alln, self.n_peaks, group=self.group)
                ld.ld_merge_peak_lists(self.allp, self.alln, self.world, self.k, self.n_rho,
                                       self.out_peaks, self.out_n, stream)
            else:
                ld.ld_merge_peak_lists(self.peaks, self.n_peaks, 1, self.k, self.n_rho,
                                       self.out_peaks, self.out_n, stream)
            self.launches += ld.ld_last_launch_count()
            mark(5)
        return self.out_peaks, self.out_n

    def vote_and_peaks(self, edges, count, stride, mark=None):
        """This rank's theta shard: vote every edge of the image (device list
        `edges`, device `count`) into rows g0 .. g1-1, then the top-k of the
        shard's own rows with global theta bins -> self.peaks, self.n_peaks."""
        ld = self.ld
        ns = max(self.g1 - self.g0, 1)
        if self.g1 > self.g0:
            # the shard's peak hint (its own keys and chunk maxima) comes with
            # the votes; the search uses the keys of the shard's own rows
            ld.ld_hough_accumulate_hint(edges, count, stride, 1, self.w, self.h, ns, self.cos_s,
                                        self.sin_s, self.acc, self.hint, self.hint_bytes, None)
            self.launches += ld.ld_last_launch_count()
        if mark:
            mark(3)
        hint = self.hint if self.g1 > self.g0 else None
        ld.ld_hough_peaks_opt(self.acc, 1, ns, self.n_rho, self.half_theta, self.half_rho,
                              self.min_votes, self.k, self.t0 - self.g0, self.t1 - self.g0,
                              self.g0, hint, self.hint_bytes if hint is not None else 0, 0,
                              self.peaks, self.n_peaks, self.ws, self.ws_bytes, None)
        self.launches += ld.ld_last_launch_count()
        if mark:
            mark(4)
