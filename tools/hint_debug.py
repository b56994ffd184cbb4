#!/usr/bin/env python
"""How good is the voting kernel's peak hint (DESIGN R25) on a workload?

    python tools/hint_debug.py cfg2 [cfg5 ...]

Votes one frame with ld_hough_accumulate_hint, then (host numpy) sorts the
hint keys, tests each against its window exactly as peaks_fused_kernel does and
prints at which sorted position the k-th verified key sits (the number of
verification rounds of PH_M keys the kernel needs), the threshold it leaves
and the frame's true k-th peak value (from the hinted search's output)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_09460_b200 import ld, synth  # noqa: E402


def main():
    for name in sys.argv[1:]:
        cfg = synth.CONFIGS[name]
        frame = synth.gen_frame(name, 0)[None]
        c, s = synth.q15_table(cfg.n_theta)
        g = torch.from_numpy(frame).cuda()
        _, edges, counts, stride = ld.sobel_binarize(g, cfg.threshold, want_binary=False)
        acc, hint = ld.hough_accumulate(edges, counts, stride, cfg.width, cfg.height, c, s,
                                        want_hint=True)
        p, n = ld.hough_peaks(acc, cfg.half_theta, cfg.half_rho, cfg.min_votes, cfg.k, hint=hint)
        A = acc[0].cpu().numpy().view(np.uint32)
        nt, nr = A.shape
        hb = hint.cpu().numpy()
        h = hb[:64].view(np.uint32)
        n_src = int(h[4]) * int(h[5])
        hdr_words = 16
        keys = hb[4 * hdr_words:4 * hdr_words + 8 * n_src].view(np.uint64)
        keys = np.sort(keys)[::-1]
        found, pos = 0, []
        for i, key in enumerate(keys):
            v = int(key >> np.uint64(32))
            idx = 0xFFFFFFFF - int(key & np.uint64(0xFFFFFFFF))
            if key == 0 or v < cfg.min_votes:
                break
            t, r = divmod(idx, nr)
            w = A[max(t - cfg.half_theta, 0):t + cfg.half_theta + 1,
                  max(r - cfg.half_rho, 0):r + cfg.half_rho + 1]
            tt, rr = np.nonzero(w == v)
            ci = (tt + max(t - cfg.half_theta, 0)) * nr + rr + max(r - cfg.half_rho, 0)
            ok = not ((w > v).any() or (ci < idx).any())
            if ok:
                found += 1
                pos.append(i)
                if found == cfg.k:
                    break
        pk = p[0].cpu().numpy()
        print("%s: header %s n_src %d keys>0 %d; k=%d verified at sorted positions %s "
              "(rounds of 32: %d); tau %s; k-th peak %d; n_peaks %d" %
              (name, h[:9].tolist(), n_src, int((keys > 0).sum()), cfg.k, pos[:70],
               pos[-1] // 32 + 1 if pos else -1,
               int(keys[pos[-1]] >> np.uint64(32)) if found == cfg.k else 0,
               int(pk[cfg.k - 1, 2]), int(n[0])))


if __name__ == "__main__":
    main()
