#!/usr/bin/env python
"""Benchmark of the lane-detection hot path (arXiv 2212.09460) on B200.

Default workload: BASELINE.json configs[2] ("cfg3"), 256 synthetic 1280x720
road frames per GPU, T=200, 180 theta bins, top-4 peaks -- the configuration
the metric "1280x720 frames/s and Hough Gvotes/s at 1/2/4/8 B200; Sobel HBM
GB/s" is quoted on.  One step = the whole hot path over the batch:
ld_sobel_binarize (fused Sobel + binarize + compaction) -> ld_hough_accumulate
(theta-band voting) -> ld_hough_peaks, each through the C ABI.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Steps go round-robin to ``--streams`` streams (default 4), each with its own
output buffers, as a serving pipeline double-buffers batches: one step's peak
search (memory-latency-bound) overlaps the next step's Sobel (issue-bound).
The headline is K such steps from a common start event to the join;
per-kernel times (and the roofline) come from the same K steps serialised on
one stream, reported next to it (``config.ms_per_step_one_stream``).

N > 1 is launched by torchrun (one process per GPU, NCCL): frames shard across
ranks with no data-path collective (weak scaling: 256 frames per rank); timing
is the max over ranks.  ``--impl reference`` times the CPU oracle (the only
"reference" this paper-only tier has) on a bounded sample of the same workload.
Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2212_09460_b200 import synth  # noqa: E402

METRIC = "1280x720 frames/s and Hough Gvotes/s at 1/2/4/8 B200; Sobel HBM GB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="cfg3", choices=list(synth.CONFIGS))
    ap.add_argument("--frames", type=int, default=None, help="frames per rank (default: config batch)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no extras)")
    ap.add_argument("--trig", default="q15", choices=["q15", "f64"],
                    help="voting table: the caller's Q15 table (the metric's) or SPEC's "
                         "float64 mode (a second workload, no peak hint)")
    ap.add_argument("--streams", type=int, default=4,
                    help="streams (each with its own buffers) the steps go to round-robin")
    ap.add_argument("--no-hint", action="store_true",
                    help="plain ld_hough_accumulate + ld_hough_peaks (no peak hint)")
    ap.add_argument("--shard", default="band", choices=["band", "theta"],
                    help="cfg5 multi-GPU decomposition: row bands + all_reduce of the "
                         "accumulator, or theta shards + all_gather of edge lists")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo: plumbing check of N ranks on fewer GPUs)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------------------
# clocks sampling during the timed region (B200_PROFILING.md recipe)
# ----------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and --impl reference)
# ----------------------------------------------------------------------------
def oracle_frames(name, first, budget_s, max_frames):
    import oracle
    cfg = synth.CONFIGS[name]
    c, s = synth.q15_table(cfg.n_theta)
    frames = []
    t_total = 0.0
    n = 0
    while n < max_frames and (t_total < budget_s or n < 2):
        img = synth.gen_frame(name, first + n)
        t0 = time.perf_counter()
        oracle.detect(img, cfg.threshold, c, s, cfg.half_theta, cfg.half_rho, cfg.min_votes,
                      cfg.k, want_binary=False, want_acc=False)
        t_total += time.perf_counter() - t0
        n += 1
        frames.append(img)
    return n, t_total


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = synth.CONFIGS[args.workload]
    per_step = max(1, min(cfg.batch, 8 if cfg.width * cfg.height <= 2_100_000 else 1))
    for i in range(args.warmup):
        oracle_frames(args.workload, i * per_step, 0.0, per_step)
    times = []
    nfr = 0
    for i in range(args.steps):
        n, t = oracle_frames(args.workload, i * per_step, 0.0, per_step)
        times.append(t)
        nfr += n
    total = sum(times)
    value = nfr / total
    sample = "%d frames of %s per step (seeds from %d), single host thread, oracle -O2" % (
        per_step, args.workload, synth.frame_seed(cfg, 0))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8/int32", "data": "synthetic",
        "config": {"workload": args.workload, "frames_per_step": per_step,
                   "width": cfg.width, "height": cfg.height, "n_theta": cfg.n_theta},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": 1, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# roofline denominators
# ----------------------------------------------------------------------------
def vote_kernel_name(c, s):
    """Which voting kernel libld.so picks for this table (label only): the
    half-angle paired kernel for a symmetric table (C[n-t] = -C[t],
    S[n-t] = S[t]) unless LD_VOTE_PAIRED=0."""
    n = len(c)
    sym = all(c[n - t] == -c[t] and s[n - t] == s[t] for t in range(1, n) if 2 * t != n)
    return ("hough_vote_pairs_kernel" if sym and os.environ.get("LD_VOTE_PAIRED") != "0"
            else "hough_vote_kernel")


def smem_atomic_peaks():
    """B5 microbenchmark (conflict-free / random / same-address red.shared.add.u32
    on all SMs), measured in this run: Gatomic/s."""
    import torch
    from paper_2212_09460_b200 import ld
    scratch = torch.empty((ld.ld_device_sm_count() * 2 * 32,), dtype=torch.int32, device="cuda")
    atom = {}
    for mode, name in ((0, "conflict_free"), (1, "random"), (2, "same_address")):
        iters = 4096 if mode < 2 else 256
        ld.ld_bench_smem_atomics(mode, iters, 1, scratch)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        n = ld.ld_bench_smem_atomics(mode, iters, 1, scratch)
        e1.record()
        torch.cuda.synchronize()
        atom[name] = n / (e0.elapsed_time(e1) / 1e3) / 1e9  # Gatomic/s
    return atom


def hbm_peak_gbs():
    """Measured HBM copy bandwidth (driver-written MEASURED_PEAKS.json), else the
    profiling guide's fallback."""
    peaks_file = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_file):
        return float(json.load(open(peaks_file)).get("hbm_gbs", 6650.0))
    return 6650.0


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------
def paper_latency(reps=50):
    """The paper's own measurement (Table 2): one 512x512 gray
    frame, pixel in -> Hough matrix (Sobel + binarize + compaction + voting,
    180 theta bins), here a synthetic cfg2-model road frame at 512x512 (the
    paper's Fig. 9 image is not available).  Device-timed medians of single
    launches: the paper's span, the span plus peaks, and the span plus peaks
    with the H2D copy of the frame and the D2H of the peaks."""
    import torch
    from paper_2212_09460_b200 import ld
    W = H = 512
    c, s = synth.q15_table(180)
    frame = synth.gen_cfg2(1, W, H)
    host = torch.from_numpy(frame[None].copy()).pin_memory()
    gray = host.cuda()
    img = ld.make_image(W, H, W, H * W, 1)
    stride = ld._round_up(H * (W - 2), 4)
    edges = torch.empty((1, stride), dtype=torch.int32, device="cuda")
    counts = torch.empty((1,), dtype=torch.int32, device="cuda")
    n_rho = 2 * ld.ld_rho_offset(W, H) + 1
    acc = torch.empty((1, 180, n_rho), dtype=torch.int32, device="cuda")
    wsb = ld.ld_hough_peaks_workspace_bytes(1, 180, n_rho, 4)
    ws = torch.empty((wsb,), dtype=torch.uint8, device="cuda")
    pk = torch.empty((1, 4, 3), dtype=torch.int32, device="cuda")
    npk = torch.empty((1,), dtype=torch.int32, device="cuda")
    pk_host = torch.empty((1, 4, 3), dtype=torch.int32).pin_memory()
    st = torch.cuda.current_stream()

    def span(peaks, copy, stream=None):
        stream = st if stream is None else stream
        if copy:
            gray.copy_(host, non_blocking=True)
        ld.ld_sobel_binarize(gray, img, 200, None, edges, stride, counts, stream)
        ld.ld_hough_accumulate(edges, counts, stride, 1, W, H, 180, c, s, acc, stream)
        if peaks:
            ld.ld_hough_peaks(acc, 1, 180, n_rho, 2, 29, 1, 4, pk, npk, ws, wsb, stream)
        if copy:
            pk_host.copy_(pk, non_blocking=True)

    out = {}
    for name, pk_on, cp in (("paper_span_ms", False, False), ("with_peaks_ms", True, False),
                            ("with_h2d_d2h_ms", True, True)):
        ts = []
        for i in range(reps + 5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            span(pk_on, cp)
            e1.record(st)
            torch.cuda.synchronize()
            if i >= 5:
                ts.append(e0.elapsed_time(e1))
        out[name] = float(np.median(ts))
    # the same two spans replayed from a CUDA graph (launch overhead removed;
    # the ABI calls are capturable: no host synchronisation inside)
    for name, pk_on in (("paper_span_graph_ms", False), ("with_peaks_graph_ms", True)):
        try:
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                span(pk_on, False, torch.cuda.current_stream())
            ts = []
            for i in range(reps + 5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(st)
                graph.replay()
                e1.record(st)
                torch.cuda.synchronize()
                if i >= 5:
                    ts.append(e0.elapsed_time(e1))
            out[name] = float(np.median(ts))
        except Exception as exc:  # capture unsupported: report why, keep the eager numbers
            out[name] = None
            out["graph_error"] = str(exc)[:200]
    out.update({"frame": "512x512 synthetic cfg2-model road frame, T=200, 180 theta",
                "edges": int(counts.item()), "paper_k80_ms": 4.874, "paper_zc706_ms": 2.62,
                "note": "context only: different hardware, image and timing span details"})
    return out


def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist
    from paper_2212_09460_b200 import ld

    # one process per GPU; with fewer GPUs than ranks (plumbing checks with the
    # gloo backend only) ranks share devices round-robin
    dev = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    cfg = synth.CONFIGS[args.workload]
    if args.workload == "cfg5":
        if args.shard == "theta":
            return run_theta(args, rank, world, local)
        return run_banded(args, rank, world, local)
    B = args.frames or cfg.batch
    W, H = cfg.width, cfg.height
    c, s = synth.q15_table(cfg.n_theta)
    first = rank * B  # weak scaling: every rank owns B frames of its own

    frames = synth.gen_batch(args.workload, first, B)
    pitch = ld._round_up(W, 16)
    host = torch.zeros((B, H, pitch), dtype=torch.uint8)
    host[:, :, :W] = torch.from_numpy(frames)
    host = host.pin_memory()
    gray = host.cuda()
    stream = torch.cuda.current_stream()

    n_rho = 2 * ld.ld_rho_offset(W, H) + 1
    img = ld.make_image(W, H, pitch, H * pitch, B)
    stride = ld._round_up(H * max(W - 2, 0), 4)
    f64 = args.trig == "f64"
    if f64:
        cf, sf = synth.f64_table(cfg.n_theta)
    use_hint = not args.no_hint and not f64
    pws_bytes = ld.ld_hough_peaks_workspace_bytes(B, cfg.n_theta, n_rho, cfg.k)
    hint_bytes = ld.ld_hough_hint_bytes(B, W, H, cfg.n_theta)

    class Buffers:
        """One step's outputs and workspaces, and the stream its steps run on."""

        def __init__(self, st):
            self.stream = st
            self.edges = torch.empty((B, stride), dtype=torch.int32, device="cuda")
            self.counts = torch.empty((B,), dtype=torch.int32, device="cuda")
            self.acc = torch.empty((B, cfg.n_theta, n_rho), dtype=torch.int32, device="cuda")
            self.pws = torch.empty((pws_bytes,), dtype=torch.uint8, device="cuda")
            self.hint = torch.empty((hint_bytes,), dtype=torch.uint8, device="cuda")
            self.peaks = torch.empty((B, cfg.k, 3), dtype=torch.int32, device="cuda")
            self.npk = torch.empty((B,), dtype=torch.int32, device="cuda")

    # steps go round-robin to `--streams` streams with a buffer set each (a
    # serving pipeline's double buffering): step i+1's Sobel can run while
    # step i's peak search still streams its accumulators
    bufs = [Buffers(stream if i == 0 else torch.cuda.Stream()) for i in range(args.streams)]
    launches = [0]

    def step(bf, ev=None):
        st = bf.stream
        if ev is not None:
            ev[0].record(st)
        ld.ld_sobel_binarize(gray, img, cfg.threshold, None, bf.edges, stride, bf.counts, st)
        launches[0] += ld.ld_last_launch_count()
        if ev is not None:
            ev[1].record(st)
        if f64:
            ld.ld_hough_accumulate_f64(bf.edges, bf.counts, stride, B, W, H, cfg.n_theta, cf, sf,
                                       bf.acc, st)
        elif use_hint:
            ld.ld_hough_accumulate_hint(bf.edges, bf.counts, stride, B, W, H, cfg.n_theta, c, s,
                                        bf.acc, bf.hint, hint_bytes, st)
        else:
            ld.ld_hough_accumulate(bf.edges, bf.counts, stride, B, W, H, cfg.n_theta, c, s,
                                   bf.acc, st)
        launches[0] += ld.ld_last_launch_count()
        if ev is not None:
            ev[2].record(st)
        if use_hint:
            ld.ld_hough_peaks_hinted(bf.acc, B, cfg.n_theta, n_rho, cfg.half_theta, cfg.half_rho,
                                     cfg.min_votes, cfg.k, bf.hint, hint_bytes, bf.peaks, bf.npk,
                                     bf.pws, pws_bytes, st)
        else:
            ld.ld_hough_peaks(bf.acc, B, cfg.n_theta, n_rho, cfg.half_theta, cfg.half_rho,
                              cfg.min_votes, cfg.k, bf.peaks, bf.npk, bf.pws, pws_bytes, st)
        launches[0] += ld.ld_last_launch_count()
        if ev is not None:
            ev[3].record(st)

    for i in range(max(args.warmup, len(bufs))):
        step(bufs[i % len(bufs)])
    torch.cuda.synchronize()
    counts, acc, peaks = bufs[0].counts, bufs[0].acc, bufs[0].peaks
    cnt = counts.cpu().numpy().astype(np.int64)
    votes = int(cnt.sum()) * cfg.n_theta
    if args.profile:
        for i in range(args.steps):
            step(bufs[0])
        torch.cuda.synchronize()
        if rank == 0:
            print(json.dumps({"profile_run": True, "votes": votes}), flush=True)
        return

    sampler = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    # (1) the headline: K steps back to back, round-robin over the streams,
    # device-timed on the launching stream from a common start to the join
    launches[0] = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_start.record(stream)
    for bf in bufs[1:]:
        bf.stream.wait_event(e_start)
    for i in range(args.steps):
        step(bufs[i % len(bufs)])
    for bf in bufs[1:]:
        j = torch.cuda.Event()
        j.record(bf.stream)
        stream.wait_event(j)
    e_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    gpu_launches = launches[0]
    elapsed_ms = float(e_start.elapsed_time(e_end))
    # (2) per-kernel times: the same K steps serialised on one stream with
    # CUDA events between the kernels (the roofline's launch durations)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    torch.cuda.synchronize()
    for i in range(args.steps):
        step(bufs[0], evs[i])
    torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    stage = np.array([[evs[i][j].elapsed_time(evs[i][j + 1]) for j in range(3)]
                      for i in range(args.steps)])  # ms
    serial_ms = float(evs[0][0].elapsed_time(evs[-1][3])) / args.steps
    for bf in bufs[1:]:  # every buffer set computed the same result
        assert torch.equal(bf.peaks, peaks) and torch.equal(bf.npk, bufs[0].npk)
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        vt = torch.tensor([votes], dtype=torch.float64, device="cuda")
        dist.all_reduce(vt, op=dist.ReduceOp.SUM)
        total_votes = float(vt.item())
    else:
        total_votes = float(votes)
    max_ms = float(t.item())
    ms_per_step = max_ms / args.steps
    frames_total = B * world
    value = frames_total / (ms_per_step / 1e3)

    # parity spot check of this run against the oracle is in tests/; here only
    # the vote-conservation invariant on the timed output (cheap, on device)
    sums = acc.view(B, -1).sum(dim=1, dtype=torch.int64).cpu().numpy()
    assert np.array_equal(sums, cnt * cfg.n_theta), "vote conservation violated"

    e2e = None
    if not args.no_e2e:
        hd = ld.HostDetector(W, H, B, cfg.n_theta, c, s, cfg.threshold, cfg.k, cfg.half_theta,
                             cfg.half_rho, cfg.min_votes, chunk_frames=32)
        for _ in range(2):
            hd(host)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            hd(host)  # synchronous: H2D of every frame, kernels, D2H of peaks/counts
        e2e_s = (time.perf_counter() - t0) / args.steps
        et = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": frames_total / float(et.item()), "unit": "frames/s",
               "h2d_bytes_per_step": B * H * pitch,
               "d2h_bytes_per_step": B * (cfg.k * 12 + 4 + 4),
               "path": "ld_detect_batch_host (pinned host frames, chunks of 32)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    atom = smem_atomic_peaks()

    sob_ms, vote_ms, peak_ms = (float(stage[:, j].mean()) for j in range(3))
    sobel_bytes = B * (W * H + 4) + 4 * int(cnt.sum())
    vote_rate = votes / (vote_ms / 1e3) / 1e9
    peaks_bytes = B * cfg.n_theta * n_rho * 4
    roofline = {"kernel": "hough_vote_f64_kernel" if f64 else vote_kernel_name(c, s),
                "bound": "smem_atomic",
                "achieved": vote_rate, "peak": atom["conflict_free"], "unit": "Gatomic/s",
                "frac": vote_rate / atom["conflict_free"], "traffic": None,
                "peak_source": "B5 microbenchmark (conflict-free red.shared.add.u32, all SMs), "
                               "measured in this run"}
    hbm_peak = hbm_peak_gbs()
    sobel_gbs = sobel_bytes / (sob_ms / 1e3) / 1e9
    cpu = None
    if not args.no_cpu_baseline and world == 1 and not f64:
        n, tcpu = oracle_frames(args.workload, 0, args.cpu_seconds, B)
        cpu = {"value": n / tcpu, "unit": "frames/s", "cores": 1, "kind": "oracle",
               "sample": "first %d frames of %s (same seeds as the GPU batch), single thread, "
                         "detect without binary/acc export" % (n, args.workload)}
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8/int32", "data": "synthetic",
        "config": {"workload": args.workload, "frames_per_gpu": B, "global_batch": frames_total,
                   "width": W, "height": H, "threshold": cfg.threshold, "n_theta": cfg.n_theta,
                   "k": cfg.k, "window": [cfg.half_theta, cfg.half_rho],
                   "parallelism": "frame-shard dp%d" % world,
                   "peak_hint": use_hint,
                   "trig": args.trig,
                   "streams": args.streams,
                   "ms_per_step_one_stream": serial_ms,
                   "l2": "inputs %.0f MB + accumulators %.0f MB per GPU exceed L2 (%.0f MB); no flush"
                         % (B * H * pitch / 1e6, peaks_bytes / 1e6, ld.ld_device_l2_bytes() / 1e6)},
        "gvotes_per_s": total_votes / (ms_per_step / 1e3) / 1e9,
        "edges_per_frame": float(cnt.mean()),
        "stages_ms": {"sobel_binarize_compact": sob_ms, "hough_vote": vote_ms,
                      "hough_peaks": peak_ms},
        "roofline": roofline,
        "roofline_sobel": {"kernel": "sobel_binarize_compact_kernel", "bound": "hbm",
                           "achieved": sobel_gbs, "peak": hbm_peak, "unit": "GB/s",
                           "frac": sobel_gbs / hbm_peak, "traffic": None,
                           "bytes_per_launch": sobel_bytes},
        "smem_atomic_peaks_gatomic_s": atom,
        "latency_512x512": paper_latency() if not args.no_e2e else None,
        "clocks": clocks,
        "gpu_launches": gpu_launches,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_banded(args, rank, world, local):
    """cfg5: one 4096^2 image in row bands over the ranks, partial accumulators
    summed by NCCL all_reduce inside the timed region (strong scaling)."""
    import torch
    import torch.distributed as dist
    from paper_2212_09460_b200 import dist as pdist
    from paper_2212_09460_b200 import ld

    cfg = synth.CONFIGS[args.workload]
    W, H = cfg.width, cfg.height
    c, s = synth.q15_table(cfg.n_theta)
    img = synth.gen_frame(args.workload, 0)  # replicated input, outside the timed region
    det = pdist.BandedDetector(W, H, cfg.n_theta, c, s, cfg.threshold, cfg.k, cfg.half_theta,
                               cfg.half_rho, cfg.min_votes, rank, world)
    det.load(img)
    stream = torch.cuda.current_stream()
    p = det.plan
    launches = [0]

    def step(ev=None):
        mark = (lambda j: ev[j].record(stream)) if ev is not None else (lambda j: None)
        mark(0)
        if p.rows > 0:
            ld.ld_sobel_binarize(det.gray, det.img, cfg.threshold, None, det.edges,
                                 det.edge_stride, det.count, stream)
            launches[0] += ld.ld_last_launch_count()
        else:
            det.count.zero_()
        mark(1)
        if det.hint is not None:  # one rank: the whole accumulator, the hint is valid
            ld.ld_hough_accumulate_hint(det.edges, det.count, det.edge_stride, 1, W, H,
                                        cfg.n_theta, c, s, det.acc, det.hint, det.hint_bytes,
                                        stream)
        else:
            ld.ld_hough_accumulate(det.edges, det.count, det.edge_stride, 1, W, H, cfg.n_theta,
                                   c, s, det.acc, stream)
        launches[0] += ld.ld_last_launch_count()
        mark(2)
        pdist.allreduce_accumulator(det.acc)
        mark(3)
        if det.hint is not None:
            ld.ld_hough_peaks_hinted(det.acc, 1, cfg.n_theta, det.n_rho, cfg.half_theta,
                                     cfg.half_rho, cfg.min_votes, cfg.k, det.hint,
                                     det.hint_bytes, det.peaks, det.n_peaks, det.ws, det.ws_bytes,
                                     stream)
        else:
            ld.ld_hough_peaks(det.acc, 1, cfg.n_theta, det.n_rho, cfg.half_theta, cfg.half_rho,
                              cfg.min_votes, cfg.k, det.peaks, det.n_peaks, det.ws, det.ws_bytes,
                              stream)
        launches[0] += ld.ld_last_launch_count()
        mark(4)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    my_edges = int(det.count.item())
    ecount = torch.tensor([my_edges], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ecount)
    edges_total = int(ecount.item())
    votes = edges_total * cfg.n_theta
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    sampler = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    launches[0] = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        step(evs[i])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    stage = np.array([[evs[i][j].elapsed_time(evs[i][j + 1]) for j in range(4)]
                      for i in range(args.steps)])
    t = torch.tensor([evs[0][0].elapsed_time(evs[-1][4])], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    # invariant on the reduced accumulator: every edge voted once per theta
    assert int(det.acc.sum(dtype=torch.int64).item()) == votes, "vote conservation violated"

    e2e = None
    if not args.no_e2e:
        host = torch.from_numpy(img[p.read_begin:p.read_end].copy()).pin_memory()
        pk_host = torch.empty((1, cfg.k, 3), dtype=torch.int32).pin_memory()
        for _ in range(2):
            det.gray[:, :W].copy_(host, non_blocking=True)
            det()
            pk_host.copy_(det.peaks, non_blocking=True)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            det.gray[:, :W].copy_(host, non_blocking=True)
            det()
            pk_host.copy_(det.peaks, non_blocking=True)
            torch.cuda.synchronize()
        et = torch.tensor([(time.perf_counter() - t0) / args.steps], dtype=torch.float64,
                          device="cuda")
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": 1.0 / float(et.item()), "unit": "frames/s",
               "h2d_bytes_per_step": int(host.numel()), "d2h_bytes_per_step": cfg.k * 12,
               "path": "band rows from pinned host -> BandedDetector -> peaks to host"}
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    atom = smem_atomic_peaks()
    sob_ms, vote_ms, ar_ms, peak_ms = (float(stage[:, j].mean()) for j in range(4))
    my_votes = my_edges * cfg.n_theta
    vote_rate = my_votes / (vote_ms / 1e3) / 1e9
    sobel_bytes = p.rows * W + 4 * my_edges + 4
    hbm = hbm_peak_gbs()
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        n, tcpu = oracle_frames(args.workload, 0, args.cpu_seconds, 1)
        cpu = {"value": n / tcpu, "unit": "frames/s", "cores": 1, "kind": "oracle",
               "sample": "the cfg5 image (seed 3), whole detect, single thread"}
    line = {
        "metric": METRIC, "value": 1e3 / ms_per_step, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u8/int32", "data": "synthetic",
        "config": {"workload": "cfg5", "width": W, "height": H, "threshold": cfg.threshold,
                   "n_theta": cfg.n_theta, "k": cfg.k, "window": [cfg.half_theta, cfg.half_rho],
                   "parallelism": "row-band x%d + %s all_reduce(SUM) of %d B" %
                                  (world, args.dist_backend.upper(), det.acc.numel() * 4),
                   "l2": "single image (16.8 MB) + acc (47.5 MB) fit in L2: latency measurement"},
        "gvotes_per_s": votes / (ms_per_step / 1e3) / 1e9,
        "edges_total": edges_total,
        "stages_ms": {"sobel_binarize_compact": sob_ms, "hough_vote": vote_ms,
                      "allreduce": ar_ms, "hough_peaks": peak_ms},
        "roofline": {"kernel": vote_kernel_name(c, s), "bound": "smem_atomic", "achieved": vote_rate,
                     "peak": atom["conflict_free"], "unit": "Gatomic/s",
                     "frac": vote_rate / atom["conflict_free"], "traffic": None,
                     "peak_source": "B5 microbenchmark measured in this run"},
        "roofline_sobel": {"kernel": "sobel_binarize_compact_kernel", "bound": "hbm",
                           "achieved": sobel_bytes / (sob_ms / 1e3) / 1e9, "peak": hbm,
                           "unit": "GB/s", "frac": sobel_bytes / (sob_ms / 1e3) / 1e9 / hbm,
                           "traffic": None, "bytes_per_launch": sobel_bytes},
        "smem_atomic_peaks_gatomic_s": atom,
        "clocks": clocks,
        "gpu_launches": launches[0],
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_theta(args, rank, world, local):
    """cfg5 theta-sharded: Sobel on the row band, edge
    lists all-gathered, every rank votes all edges into its theta shard (+halo
    rows), peaks of its own rows, top-k lists all-gathered and merged on the
    device.  Strong scaling; the result is identical on every rank."""
    import torch
    import torch.distributed as dist
    from paper_2212_09460_b200 import dist as pdist

    cfg = synth.CONFIGS[args.workload]
    W, H = cfg.width, cfg.height
    c, s = synth.q15_table(cfg.n_theta)
    img = synth.gen_frame(args.workload, 0)
    det = pdist.ThetaShardedDetector(W, H, cfg.n_theta, c, s, cfg.threshold, cfg.k,
                                     cfg.half_theta, cfg.half_rho, cfg.min_votes, rank, world)
    det.load(img)
    stream = torch.cuda.current_stream()
    launches = [0]

    def step(ev=None):
        det((lambda j: ev[j].record(stream)) if ev is not None else None)
        launches[0] += det.launches

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    my_edges = int(det.band.count.item())
    ecount = torch.tensor([my_edges], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ecount)
    edges_total = int(ecount.item())
    votes = edges_total * cfg.n_theta
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    sampler = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    launches[0] = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        step(evs[i])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    stage = np.array([[evs[i][j].elapsed_time(evs[i][j + 1]) for j in range(5)]
                      for i in range(args.steps)])
    t = torch.tensor([evs[0][0].elapsed_time(evs[-1][5])], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    # invariant on the shard accumulator: every edge voted once per slice row
    slice_rows = det.g1 - det.g0
    assert int(det.acc.sum(dtype=torch.int64).item()) == edges_total * slice_rows, \
        "vote conservation violated"

    e2e = None
    if not args.no_e2e:
        p = det.band.plan
        host = torch.from_numpy(img[p.read_begin:p.read_end].copy()).pin_memory()
        pk_host = torch.empty((1, cfg.k, 3), dtype=torch.int32).pin_memory()
        times = []
        for i in range(args.steps + 2):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            det.band.gray[:, :W].copy_(host, non_blocking=True)
            pk, _ = det()
            pk_host.copy_(pk, non_blocking=True)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        et = torch.tensor([sum(times[2:]) / args.steps], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": 1.0 / float(et.item()), "unit": "frames/s",
               "h2d_bytes_per_step": int(host.numel()), "d2h_bytes_per_step": cfg.k * 12,
               "path": "band rows from pinned host -> ThetaShardedDetector -> peaks to host"}
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    atom = smem_atomic_peaks()
    sob_ms, xch_ms, vote_ms, peak_ms, merge_ms = (float(stage[:, j].mean()) for j in range(5))
    my_votes = edges_total * slice_rows
    vote_rate = my_votes / (vote_ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": 1e3 / ms_per_step, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u8/int32", "data": "synthetic",
        "config": {"workload": "cfg5", "width": W, "height": H, "threshold": cfg.threshold,
                   "n_theta": cfg.n_theta, "k": cfg.k, "window": [cfg.half_theta, cfg.half_rho],
                   "parallelism": "theta-shard x%d (+%d halo rows) + %s all_gather of edge lists"
                                  % (world, cfg.half_theta, args.dist_backend.upper()),
                   "l2": "single image (16.8 MB) + acc slice fit in L2: latency measurement"},
        "gvotes_per_s": votes / (ms_per_step / 1e3) / 1e9,
        "edges_total": edges_total,
        "stages_ms": {"sobel_binarize_compact": sob_ms, "edge_allgather": xch_ms,
                      "hough_vote": vote_ms, "hough_peaks": peak_ms, "topk_merge": merge_ms},
        "roofline": {"kernel": vote_kernel_name(det.cos_s, det.sin_s), "bound": "smem_atomic", "achieved": vote_rate,
                     "peak": atom["conflict_free"], "unit": "Gatomic/s",
                     "frac": vote_rate / atom["conflict_free"], "traffic": None,
                     "peak_source": "B5 microbenchmark measured in this run"},
        "smem_atomic_peaks_gatomic_s": atom,
        "clocks": clocks,
        "gpu_launches": launches[0],
        "e2e": e2e,
        "cpu_baseline": None,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
