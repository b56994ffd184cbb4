#!/usr/bin/env python
"""Per-frame phase clocks of peaks_fused_kernel (a -DLD_PF_STATS=1 build named
by LD_LIB): bound / sparse cycles, hot chunks, prefilter survivors, candidates.

    LD_LIB=build/variants/libld_pfstats.so python tools/pf_stats.py cfg3
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_09460_b200 import ld, synth  # noqa: E402


def main():
    for name in sys.argv[1:]:
        cfg = synth.CONFIGS[name]
        nf = min(cfg.batch, 16)
        frames = synth.gen_batch(name, 0, nf) if cfg.batch > 1 else synth.gen_frame(name, 0)[None]
        c, s = synth.q15_table(cfg.n_theta)
        g = torch.from_numpy(frames).cuda()
        _, edges, counts, stride = ld.sobel_binarize(g, cfg.threshold, want_binary=False)
        acc, hint = ld.hough_accumulate(edges, counts, stride, cfg.width, cfg.height, c, s,
                                        want_hint=True)
        b, nt, nr = acc.shape
        wsb = ld.ld_hough_peaks_workspace_bytes(b, nt, nr, cfg.k)
        ws = torch.zeros((wsb,), dtype=torch.uint8, device="cuda")
        pk = torch.empty((b, cfg.k, 3), dtype=torch.int32, device="cuda")
        npk = torch.empty((b,), dtype=torch.int32, device="cuda")
        ld.ld_hough_peaks_hinted(acc, b, nt, nr, cfg.half_theta, cfg.half_rho, cfg.min_votes,
                                 cfg.k, hint, hint.numel(), pk, npk, ws, wsb)
        torch.cuda.synchronize()
        head = (4 * b + 255) // 256 * 256
        cand = ws[2 * head:].cpu().numpy()[:8 * 16 * b].view(np.uint64).reshape(b, 16)
        res = ws[head:head + 4 * b].cpu().numpy().view(np.uint32)
        print(name, "cycles bound-sort/verify/sparse, hot, survivors, cand, rounds, n_src, tau, load-cycles, 1-load latency, window-test cycles, resolved")
        for f in range(b):
            print("  ", cand[f, :12].tolist(), int(res[f]))


if __name__ == "__main__":
    main()
