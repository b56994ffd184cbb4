"""Experiment: throughput of back-to-back cfg3 steps on 1 stream vs N streams
(each stream its own buffer set, steps assigned round-robin), so that one
step's peak search can overlap the next step's Sobel."""
import os
import sys
import time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_09460_b200 import ld, synth  # noqa: E402

cfg = synth.CONFIGS["cfg3"]
B, W, H = cfg.batch, cfg.width, cfg.height
c, s = synth.q15_table(cfg.n_theta)
pitch = ld._round_up(W, 16)
g = torch.zeros((B, H, pitch), dtype=torch.uint8)
g[:, :, :W] = torch.from_numpy(synth.gen_batch("cfg3", 0, B))
gray = g.cuda()
img = ld.make_image(W, H, pitch, H * pitch, B)
n_rho = 2 * ld.ld_rho_offset(W, H) + 1
stride = ld._round_up(H * (W - 2), 4)


class Bufs:
    def __init__(self):
        self.edges = torch.empty((B, stride), dtype=torch.int32, device="cuda")
        self.counts = torch.empty((B,), dtype=torch.int32, device="cuda")
        self.acc = torch.empty((B, cfg.n_theta, n_rho), dtype=torch.int32, device="cuda")
        self.pwb = ld.ld_hough_peaks_workspace_bytes(B, cfg.n_theta, n_rho, cfg.k)
        self.pws = torch.empty((self.pwb,), dtype=torch.uint8, device="cuda")
        self.hb = ld.ld_hough_hint_bytes(B, W, H, cfg.n_theta)
        self.hint = torch.empty((self.hb,), dtype=torch.uint8, device="cuda")
        self.peaks = torch.empty((B, cfg.k, 3), dtype=torch.int32, device="cuda")
        self.npk = torch.empty((B,), dtype=torch.int32, device="cuda")
        self.stream = torch.cuda.Stream()


def step(b):
    st = b.stream
    ld.ld_sobel_binarize(gray, img, cfg.threshold, None, b.edges, stride, b.counts, st)
    ld.ld_hough_accumulate_hint(b.edges, b.counts, stride, B, W, H, cfg.n_theta, c, s, b.acc,
                                b.hint, b.hb, st)
    ld.ld_hough_peaks_hinted(b.acc, B, cfg.n_theta, n_rho, cfg.half_theta, cfg.half_rho,
                             cfg.min_votes, cfg.k, b.hint, b.hb, b.peaks, b.npk, b.pws, b.pwb, st)


bufs = [Bufs() for _ in range(3)]
for ns in (1, 2, 3):
    for i in range(6):
        step(bufs[i % ns])
    torch.cuda.synchronize()
    K = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main = torch.cuda.current_stream()
    e0.record(main)
    for b in bufs[:ns]:
        b.stream.wait_event(e0)
    for i in range(K):
        step(bufs[i % ns])
    for b in bufs[:ns]:
        ev = torch.cuda.Event()
        ev.record(b.stream)
        main.wait_event(ev)
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    ref = bufs[0].peaks.clone()
    print({"streams": ns, "ms_per_step": round(ms, 4), "frames_per_s": round(B / ms * 1e3)})
    for b in bufs[1:ns]:
        assert torch.equal(b.peaks, ref)
