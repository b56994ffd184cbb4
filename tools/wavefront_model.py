"""Model of the voting kernel's shared-memory wavefronts per vote instruction
for a given edge-list order.

Measured cost model of ATOMS on B200 (tools/atoms_probe.cu): a warp's 32
votes into one accumulator row cost as many wavefronts as the largest number
of DISTINCT counters that share a bank (same-counter lanes merge for free).
The voting kernel gives lane l of a warp the list entries blk + 32 j + l, so
every aligned window of 32 consecutive list entries is one ATOMS per row.
This script rebuilds B1's emission order on a cfg3 frame (a column-major or
snake walk of each warp's 16 x 8-pixel blocks, slices in random order) and
reports the mean wavefronts per ATOMS over all 180 rows.  CPU only:

    python tools/wavefront_model.py
"""
import os
import sys

import math

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_09460_b200 import synth  # noqa: E402


def binarize(img, threshold):
    """|Gx| + |Gy| >= T with a zero 1-px border (DESIGN R1-R6), numpy, for the
    model frame only (not a checker: the oracle is oracle/)."""
    p = img.astype(np.int32)
    gx = (p[:-2, 2:] + 2 * p[1:-1, 2:] + p[2:, 2:]) - (p[:-2, :-2] + 2 * p[1:-1, :-2] + p[2:, :-2])
    gy = (p[2:, :-2] + 2 * p[2:, 1:-1] + p[2:, 2:]) - (p[:-2, :-2] + 2 * p[:-2, 1:-1] + p[:-2, 2:])
    out = np.zeros(img.shape, bool)
    out[1:-1, 1:-1] = (np.abs(gx) + np.abs(gy)) >= threshold
    return out


def wavefronts(edges, width, height, n_theta):
    c, s = synth.q15_table(n_theta)
    d = math.isqrt(width * width + height * height - 1) + 1
    n = len(edges) // 32 * 32
    x = (edges[:n] & 0xFFFF).reshape(-1, 32)
    y = (edges[:n] >> 16).reshape(-1, 32)
    tot = cnt = 0
    rows = np.repeat(np.arange(x.shape[0]), 32).reshape(-1, 32)
    for t in range(n_theta):
        b = np.sort(((x * int(c[t]) + y * int(s[t]) + (1 << 14)) >> 15) + d, axis=1)
        uniq = np.concatenate([np.ones((b.shape[0], 1), bool), b[:, 1:] != b[:, :-1]], axis=1)
        m = np.zeros((b.shape[0], 32), np.int32)
        np.add.at(m, (rows[uniq], (b % 32)[uniq]), 1)
        tot += m.max(axis=1).sum()
        cnt += b.shape[0]
    return tot / cnt


def b1_order(binary, snake, seed=0, th=128, tw=224, sr=8):
    """The list order of ld_sobel.cu: per tile and warp, the warp's 32 blocks
    chunk by chunk (strips down, or alternately down/up with snake), rows top
    to bottom, highest/lowest set bit alternating; slices in random order."""
    h, w = binary.shape
    slices = []
    for ty in range(0, h, th):
        for tx in range(0, w, tw):
            for wp in range(7):
                def key(t):
                    c, st = t % 14, t // 14
                    return c * 1000 + (100 - st if snake and c % 2 else st)
                sl = []
                for t in sorted(range(32 * wp, 32 * wp + 32), key=key):
                    chunk, strip = t % 14, t // 14
                    xs, yb = tx + 16 * chunk, ty + sr * strip
                    for i in range(sr):
                        yy = yb + i
                        if yy >= h or xs >= w:
                            continue
                        bits = list(np.flatnonzero(binary[yy, xs:xs + 16]))
                        lo, hi = 0, len(bits) - 1
                        while lo <= hi:
                            sl.append((yy << 16) | (xs + bits[hi]))
                            if hi != lo:
                                sl.append((yy << 16) | (xs + bits[lo]))
                            hi -= 1
                            lo += 1
                slices.append(sl)
    order = np.random.default_rng(seed).permutation(len(slices))
    return np.array([e for i in order for e in slices[i]], dtype=np.int64)


if __name__ == "__main__":
    img = synth.gen_frame("cfg3", 0)
    binary = binarize(img, 200)
    for snake in (False, True):
        e = b1_order(binary, snake)
        print("snake=%s: %.3f wavefronts per ATOMS" % (snake, wavefronts(e, 1280, 720, 180)))
