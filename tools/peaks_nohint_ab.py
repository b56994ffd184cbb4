#!/usr/bin/env python
"""Unhinted peak search on a voted accumulator: the default path (hint taken
from the accumulator, then the fused search) against the dense kernels alone
(LD_PEAKS_DENSE).  Mean ms over --reps serialised calls (CUDA events).

    python tools/peaks_nohint_ab.py cfg2 cfg3 cfg4 cfg5
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_09460_b200 import ld, synth  # noqa: E402


def main():
    for name in sys.argv[1:]:
        cfg = synth.CONFIGS[name]
        frames = synth.gen_batch(name, 0, cfg.batch) if cfg.batch > 1 else synth.gen_frame(name, 0)[None]
        c, s = synth.q15_table(cfg.n_theta)
        g = torch.from_numpy(frames).cuda()
        _, edges, counts, stride = ld.sobel_binarize(g, cfg.threshold, want_binary=False)
        acc = ld.hough_accumulate(edges, counts, stride, cfg.width, cfg.height, c, s)
        out = {"workload": name}
        for label, flags in (("default", 0), ("dense", ld.LD_PEAKS_DENSE)):
            ts = []
            for i in range(13):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                p, n = ld.hough_peaks(acc, cfg.half_theta, cfg.half_rho, cfg.min_votes, cfg.k,
                                      flags=flags)
                e1.record()
                torch.cuda.synchronize()
                if i >= 3:
                    ts.append(e0.elapsed_time(e1))
            out[label + "_ms"] = sum(ts) / len(ts)
            out[label + "_sum"] = int(p.sum().item())
        print(json.dumps(out))


if __name__ == "__main__":
    main()
