"""Frame-by-frame parity of a batch of GPU outputs against the CPU oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): used by tests/ and by the
cpu_baseline leg of bench.py, which runs the oracle over the very frames the
timed GPU steps processed and compares every one of them.  No arithmetic of
the method lives here: each frame goes through ``oracle.detect`` (the C
oracle, ld_oracle.c) and the GPU's outputs for that frame are compared with
exact equality -- edge count, edge list as a set (DESIGN R15), accumulator,
peaks (DESIGN R22).
"""
from __future__ import annotations

import time

import numpy as np

from . import detect, host_cores, map_frames


def _peaks_list(p):
    p = np.asarray(p)
    if p.dtype.names:
        return [(int(a), int(b), int(c)) for a, b, c in
                zip(p["theta_bin"], p["rho_bin"], p["votes"])]
    p = p.reshape(-1, 3)
    return [(int(a), int(b), int(np.uint32(np.int32(c)))) for a, b, c in p]


def compare_frame(frame, threshold, cos_q15, sin_q15, half_theta, half_rho, min_votes, k,
                  count, peaks, n_peaks, acc=None, edges=None, r=None):
    """Run the oracle on one frame (unless its result r is given) and compare;
    returns None if identical, else a one-line description of the first
    difference."""
    if r is None:
        r = detect(frame, threshold, cos_q15, sin_q15, half_theta, half_rho, min_votes, k,
                   want_binary=False, want_acc=acc is not None)
    if int(count) != r["n_edges"]:
        return "edge count %d != oracle %d" % (int(count), r["n_edges"])
    if edges is not None:
        got = np.sort(np.asarray(edges, dtype=np.uint32))
        if not np.array_equal(got, r["edges"]):  # oracle emits raster = ascending order
            bad = int(np.flatnonzero(got != r["edges"])[0])
            return "edge set differs at sorted index %d" % bad
    if acc is not None:
        a = np.asarray(acc).view(np.uint32).reshape(r["acc"].shape)
        if not np.array_equal(a, r["acc"]):
            t, rr = np.argwhere(a != r["acc"])[0]
            return "acc[%d][%d] = %d != oracle %d" % (t, rr, a[t, rr], r["acc"][t, rr])
    if int(n_peaks) != r["n_peaks"]:
        return "n_peaks %d != oracle %d" % (int(n_peaks), r["n_peaks"])
    got = _peaks_list(peaks)[: max(int(n_peaks), 0)]
    want = _peaks_list(r["peaks"])[: r["n_peaks"]]
    if got != want:
        return "peaks %s != oracle %s" % (got, want)
    # unused slots hold the sentinel {-1, -1, 0}
    rest = _peaks_list(peaks)[max(int(n_peaks), 0):]
    if any(p != (-1, -1, 0) for p in rest):
        return "unused peak slot is not the sentinel"
    return None


def check_batch(frames, threshold, cos_q15, sin_q15, half_theta, half_rho, min_votes, k,
                get, workers: int | None = None) -> dict:
    """Compare every frame.  frames: uint8 [B][H][W]; get(f) returns the GPU's
    (count, peaks, n_peaks, acc_or_None, edges_or_None) for frame f (host
    arrays).  Returns {frames, ok, mismatches, first_mismatch, seconds,
    workers}; the oracle work is frame-parallel over `workers` threads."""
    n = len(frames)
    workers = workers or host_cores()

    def one(f):
        count, peaks, n_peaks, acc, edges = get(f)
        t = time.perf_counter()
        r = detect(frames[f], threshold, cos_q15, sin_q15, half_theta, half_rho, min_votes, k,
                   want_binary=False, want_acc=acc is not None)
        t = time.perf_counter() - t
        why = compare_frame(frames[f], threshold, cos_q15, sin_q15, half_theta, half_rho,
                            min_votes, k, count, peaks, n_peaks, acc, edges, r)
        return t, (None if why is None else (f, why))

    t0 = time.perf_counter()
    out = map_frames(one, range(n), workers)
    dt = time.perf_counter() - t0
    res = [m for _, m in out if m is not None]
    return {"frames": n, "ok": not res, "mismatches": len(res),
            "first_mismatch": None if not res else "frame %d: %s" % res[0],
            "seconds": dt, "oracle_thread_seconds": sum(t for t, _ in out),
            "workers": workers}
