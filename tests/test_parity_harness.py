"""The frame-parallel parity harness (oracle/parity.py) itself, on CPU: it
accepts the oracle's own outputs and reports each kind of difference (count,
edge set, accumulator, peaks, sentinel) as the first mismatch, in order."""
import numpy as np
import pytest

from paper_2212_09460_b200 import synth


@pytest.fixture(scope="module")
def case(oracle):
    cfg = synth.CONFIGS["cfg1"]
    c, s = synth.q15_table(cfg.n_theta)
    frames = np.stack([synth.gen_frame("cfg1", 0), synth.random_image(5, 320, 240, "uniform")])
    outs = [oracle.detect(f, cfg.threshold, c, s, cfg.half_theta, cfg.half_rho, cfg.min_votes,
                          cfg.k, want_binary=False) for f in frames]
    return cfg, c, s, frames, outs


def _gpu_like(out, k):
    """The oracle's result in the GPU's host layout (int32 [k][3], sentinel fill)."""
    pk = np.full((k, 3), -1, np.int32)
    pk[:, 2] = 0
    for i in range(out["n_peaks"]):
        p = out["peaks"][i]
        pk[i] = (p["theta_bin"], p["rho_bin"], np.int32(np.uint32(p["votes"]).view(np.int32)))
    return pk


def _run(oracle, case, mutate=None, workers=2):
    from oracle import parity
    cfg, c, s, frames, outs = case

    def get(f):
        o = outs[f]
        cnt, pk, npk = o["n_edges"], _gpu_like(o, cfg.k), o["n_peaks"]
        acc, edges = o["acc"].copy(), o["edges"][::-1].copy()  # any order: a set
        if mutate and f == 1:
            cnt, pk, npk, acc, edges = mutate(cnt, pk, npk, acc, edges)
        return cnt, pk, npk, acc, edges

    return parity.check_batch(frames, cfg.threshold, c, s, cfg.half_theta, cfg.half_rho,
                              cfg.min_votes, cfg.k, get, workers=workers)


def test_identical_outputs_pass(oracle, case):
    r = _run(oracle, case)
    assert r["ok"] and r["frames"] == 2 and r["first_mismatch"] is None
    assert r["oracle_thread_seconds"] > 0


def test_count_mismatch(oracle, case):
    r = _run(oracle, case, lambda c, p, n, a, e: (c + 1, p, n, a, e))
    assert not r["ok"] and r["first_mismatch"].startswith("frame 1: edge count")


def test_edge_set_mismatch(oracle, case):
    def m(c, p, n, a, e):
        e = e.copy()
        e[0] ^= 1
        return c, p, n, a, e
    r = _run(oracle, case, m)
    assert "edge set" in r["first_mismatch"]


def test_acc_mismatch(oracle, case):
    def m(c, p, n, a, e):
        a = a.copy()
        a[3, 7] += 1
        return c, p, n, a, e
    r = _run(oracle, case, m)
    assert "acc[3][7]" in r["first_mismatch"]


def test_peak_and_sentinel_mismatch(oracle, case):
    def swap(c, p, n, a, e):
        p = p.copy()
        p[0, 1] += 1
        return c, p, n, a, e
    assert "peaks" in _run(oracle, case, swap)["first_mismatch"]

    def bad_sentinel(c, p, n, a, e):
        p = p.copy()
        p[-1] = (5, 5, 5)
        return c, p, min(n, p.shape[0] - 1), a, e
    r = _run(oracle, case, bad_sentinel)
    assert not r["ok"]


def test_map_frames_order_and_cores(oracle):
    assert oracle.map_frames(lambda i: i * i, range(10), 3) == [i * i for i in range(10)]
    assert oracle.host_cores() >= 1 and isinstance(oracle.cpu_model(), str)
