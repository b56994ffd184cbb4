"""Pins of the CPU oracle against values the paper and mathematics fix (CPU only).

Each test pins one oracle function to something other than itself: a
hand-computed value (tests/golden, each with its citation), a closed form, a
library routine (scipy / numpy), exact rational arithmetic, an invariant, or
brute force on tiny inputs.  DESIGN.md section 4 maps every pin to the paper.
"""
from fractions import Fraction
import itertools
import math

import numpy as np
import pytest
from scipy import signal

from conftest import load_golden
from paper_2212_09460_b200 import synth

SX = np.array([[-1, 0, 1], [-2, 0, 2], [-1, 0, 1]])   # Fig. 2
SY = np.array([[1, 2, 1], [0, 0, 0], [-1, -2, -1]])


# ----------------------------------------------------------------------------
# Geometry (DESIGN R10)
# ----------------------------------------------------------------------------
def test_rho_offset_golden(oracle):
    g = load_golden("geometry_pins.json")
    for case in g["rho_offset"]:
        assert oracle.rho_offset(case["w"], case["h"]) == case["D"], case
    for case in g["acc_bytes"]:
        d = oracle.rho_offset(case["w"], case["h"])
        assert case["n_theta"] * (2 * d + 1) * 4 == case["bytes"], case


def test_rho_offset_is_ceil_sqrt(oracle):
    # math.isqrt is an exact library integer square root
    rng = np.random.default_rng(5)
    for w, h in list(rng.integers(1, 16385, size=(300, 2))) + [(1, 1), (16384, 16384)]:
        s = int(w) ** 2 + int(h) ** 2
        r = math.isqrt(s)
        want = r if r * r == s else r + 1
        assert oracle.rho_offset(int(w), int(h)) == want


# ----------------------------------------------------------------------------
# Sobel + binarize (Eq. 1, Fig. 2; DESIGN R1-R4)
# ----------------------------------------------------------------------------
def test_sobel_hand_computed_centres(oracle):
    g = load_golden("sobel_pins.json")
    for case in g["center_cases"]:
        img = np.array(case["image"], np.uint8)
        assert oracle.sobel_magnitude(img)[1, 1] == case["center"], case["cite"]


def test_sobel_step_and_ramp(oracle):
    g = load_golden("sobel_pins.json")
    st = g["step_4x6"]
    img = np.array(st["image"], np.uint8)
    mag = oracle.sobel_magnitude(img)
    assert mag[1:-1, 1:-1].tolist() == st["magnitude_interior"]
    b = oracle.sobel_binarize(img, st["threshold"])
    assert int((b == 255).sum()) == st["edges"]
    rp = g["ramp_4x5"]
    img = np.array(rp["image"], np.uint8)
    assert oracle.sobel_magnitude(img)[1:-1, 1:-1].tolist() == rp["magnitude_interior"]
    for t, e in rp["thresholds"]:
        assert int((oracle.sobel_binarize(img, t) == 255).sum()) == e


def test_sobel_maximum_is_1530_and_threshold_edges(oracle):
    img = np.array([[0, 255, 255], [0, 0, 255], [0, 0, 0]], np.uint8)
    assert oracle.sobel_binarize(img, 1530)[1, 1] == 255
    assert oracle.sobel_binarize(img, 1531)[1, 1] == 0


def test_sobel_matches_scipy_correlate(oracle):
    # Library routine: scipy 2-D correlation ('valid' = interior) with Fig. 2.
    for seed, (h, w) in enumerate([(3, 3), (7, 11), (40, 33), (64, 64)]):
        img = synth.random_image(seed, w, h)
        gx = signal.correlate2d(img.astype(np.int64), SX, mode="valid")
        gy = signal.correlate2d(img.astype(np.int64), SY, mode="valid")
        mag = oracle.sobel_magnitude(img)
        assert np.array_equal(mag[1:-1, 1:-1], np.abs(gx) + np.abs(gy))
        # convolution (180-degree flipped kernels) gives the same |G| (DESIGN R1)
        cx = signal.convolve2d(img.astype(np.int64), SX, mode="valid")
        cy = signal.convolve2d(img.astype(np.int64), SY, mode="valid")
        assert np.array_equal(mag[1:-1, 1:-1], np.abs(cx) + np.abs(cy))


# ----------------------------------------------------------------------------
# NEXT 4: the paper's zero-padded border and SPEC's 8-bit clamp
# (S:111-116); DESIGN R23, R24
# ----------------------------------------------------------------------------
def test_zero_pad_hand_computed(oracle):
    # all-255 3x3, zero-padded: corners see 4 bright pixels, edge midpoints 6
    img = np.full((3, 3), 255, np.uint8)
    mag = oracle.sobel_magnitude_ex(img, oracle.ZERO_PAD)
    assert mag.tolist() == [[1530, 1020, 1530], [1020, 0, 1020], [1530, 1020, 1530]]
    # a single pixel surrounded by padding: Gx = Gy = 0
    assert oracle.sobel_magnitude_ex(np.array([[200]], np.uint8), oracle.ZERO_PAD)[0, 0] == 0
    # 1 x 3 row [0, 0, 255]: the middle pixel sees +255 twice in Gx (rows -1, +1 are 0)
    row = np.array([[0, 0, 255]], np.uint8)
    assert oracle.sobel_magnitude_ex(row, oracle.ZERO_PAD)[0, 1] == 2 * 255


def test_zero_pad_matches_scipy_constant_mode(oracle):
    # library routine: scipy correlation over the zero-padded image ('same'
    # output, fill value 0) with the Fig. 2 kernels, every pixel incl. borders
    for seed, (h, w) in enumerate([(1, 1), (1, 7), (2, 2), (3, 5), (17, 9), (40, 33)]):
        img = synth.random_image(100 + seed, w, h).astype(np.int64)
        gx = signal.correlate2d(img, SX, mode="same", boundary="fill", fillvalue=0)
        gy = signal.correlate2d(img, SY, mode="same", boundary="fill", fillvalue=0)
        mag = oracle.sobel_magnitude_ex(img.astype(np.uint8), oracle.ZERO_PAD)
        assert np.array_equal(mag, np.abs(gx) + np.abs(gy)), (h, w)
        # interior identical to the forced-zero-border magnitude
        assert np.array_equal(mag[1:-1, 1:-1], oracle.sobel_magnitude(img.astype(np.uint8))[1:-1, 1:-1])


def test_clamp_and_flag_combinations(oracle):
    img = synth.random_image(5, 50, 31)
    for t in (-3, 0, 1, 200, 255):
        # clamping to 255 cannot change a ">= T" decision for T <= 255
        assert np.array_equal(oracle.sobel_binarize_ex(img, t, oracle.CLAMP_255),
                              oracle.sobel_binarize(img, t))
        assert np.array_equal(oracle.sobel_binarize_ex(img, t, oracle.CLAMP_255 | oracle.ZERO_PAD),
                              oracle.sobel_binarize_ex(img, t, oracle.ZERO_PAD))
    for t in (256, 1000, 1530):  # above the clamp nothing passes
        assert not oracle.sobel_binarize_ex(img, t, oracle.CLAMP_255).any()
        assert not oracle.sobel_binarize_ex(img, t, oracle.CLAMP_255 | oracle.ZERO_PAD).any()
    assert np.array_equal(oracle.sobel_binarize_ex(img, 200, 0), oracle.sobel_binarize(img, 200))
    zp = oracle.sobel_binarize_ex(img, 200, oracle.ZERO_PAD)
    mag = oracle.sobel_magnitude_ex(img, oracle.ZERO_PAD)
    assert np.array_equal(zp == 255, mag >= 200)


def test_sobel_exhaustive_binary_patches(oracle):
    # every {0,255}^9 patch: |G| even, <= 1530, max attained; matches the literal sum
    mags = []
    for bits in range(512):
        p = np.array([(bits >> i) & 1 for i in range(9)], np.int64).reshape(3, 3) * 255
        m = int(oracle.sobel_magnitude(p.astype(np.uint8))[1, 1])
        assert m == abs(int((SX * p).sum())) + abs(int((SY * p).sum()))
        mags.append(m)
    assert max(mags) == 1530 and all(m % 2 == 0 for m in mags)


def test_sobel_border_and_tiny_images(oracle):
    for h, w in [(1, 1), (1, 7), (2, 2), (2, 9), (9, 2), (3, 3), (5, 4)]:
        img = synth.random_image(h * 31 + w, w, h, "binary")
        b = oracle.sobel_binarize(img, 0)
        assert b[0, :].max(initial=0) == 0 and b[-1, :].max(initial=0) == 0
        assert b[:, 0].max(initial=0) == 0 and b[:, -1].max(initial=0) == 0
        # T <= 0: every interior pixel is an edge
        assert int((b == 255).sum()) == max(h - 2, 0) * max(w - 2, 0)


def test_sobel_flip_invariance_and_monotone_threshold(oracle):
    img = synth.random_image(11, 37, 29)
    base = oracle.sobel_binarize(img, 200)
    assert np.array_equal(oracle.sobel_binarize(img[:, ::-1], 200), base[:, ::-1])
    assert np.array_equal(oracle.sobel_binarize(img[::-1, :], 200), base[::-1, :])
    sq = synth.random_image(12, 31, 31)
    assert np.array_equal(oracle.sobel_binarize(sq.T, 150), oracle.sobel_binarize(sq, 150).T)
    counts = [int((oracle.sobel_binarize(img, t) == 255).sum()) for t in range(0, 1600, 97)]
    assert all(a >= b for a, b in zip(counts, counts[1:]))


def test_constant_image_has_no_edges(oracle):
    for v in (0, 77, 255):
        img = np.full((13, 17), v, np.uint8)
        assert (oracle.sobel_binarize(img, 1) == 0).all()


# ----------------------------------------------------------------------------
# Compaction
# ----------------------------------------------------------------------------
def test_compact_matches_numpy_nonzero(oracle):
    for seed, (h, w) in enumerate([(1, 1), (5, 9), (33, 70)]):
        b = synth.random_image(seed, w, h, "binary")
        ys, xs = np.nonzero(b == 255)  # library: row-major order
        want = (ys.astype(np.uint32) << 16) | xs.astype(np.uint32)
        assert np.array_equal(oracle.compact(b), want)


# ----------------------------------------------------------------------------
# Trig table input pins (the table is an input, DESIGN R11)
# ----------------------------------------------------------------------------
def test_q15_table_pins():
    g = load_golden("hough_pins.json")
    for case in g["q15"]:
        n = case["n_theta"]
        c, s = synth.q15_table(n)
        assert c[0] == case["C0"] and s[n // 2] == case["S_half"] and c[n // 2] == case["C_half"]
        assert c[n // 4] == case["C_quarter"] and s[n // 4] == case["S_quarter"]
        for t in range(1, n):  # Eq. 4-5 hold exactly
            assert s[t] == s[n - t] and c[t] == -c[n - t]
        th = np.pi * np.arange(n) / n
        assert np.abs(c - 32768 * np.cos(th)).max() <= 0.5
        assert np.abs(s - 32768 * np.sin(th)).max() <= 0.5


# ----------------------------------------------------------------------------
# Hough voting (Eq. 3; DESIGN R8-R12)
# ----------------------------------------------------------------------------
def _round_half_up(fr: Fraction) -> int:
    return math.floor(fr + Fraction(1, 2))


@pytest.mark.parametrize("n_theta", [1, 2, 3, 8, 180, 181, 720, 1024])
def test_single_pixel_exact_rational(oracle, n_theta):
    # One pixel votes once per theta at round_half_up((x C + y S) / 2^15) + D,
    # computed with exact rationals (no shifts, no floor_div).
    c, s = synth.q15_table(n_theta)
    w, h = 97, 61
    d = oracle.rho_offset(w, h)
    rng = np.random.default_rng(n_theta)
    pts = [(0, 0), (w - 1, h - 1), (w - 1, 0), (0, h - 1)] + \
        [tuple(map(int, p)) for p in zip(rng.integers(0, w, 6), rng.integers(0, h, 6))]
    for x, y in pts:
        acc = oracle.hough_accumulate(np.array([(y << 16) | x], np.uint32), w, h, c, s)
        assert int(acc.sum()) == n_theta
        for t in range(n_theta):
            r = _round_half_up(Fraction(x * int(c[t]) + y * int(s[t]), 32768))
            assert acc[t, r + d] == 1
            # Eq. 3 error bound: |r - (x cos + y sin)| <= 1/2 + (x + y) / 2^16
            true_r = x * math.cos(math.pi * t / n_theta) + y * math.sin(math.pi * t / n_theta)
            assert abs(r - true_r) <= 0.5 + (x + y) / 65536.0 + 1e-9


def test_origin_votes_at_D(oracle):
    c, s = synth.q15_table(180)
    acc = oracle.hough_accumulate(np.array([0], np.uint32), 320, 240, c, s)
    assert (acc[:, 400] == 1).all() and int(acc.sum()) == 180


def test_rho_of_spec_examples(oracle):
    c, s = synth.q15_table(180)
    d = 400
    acc = oracle.hough_accumulate(np.array([(7 << 16) | 10], np.uint32), 320, 240, c, s)
    assert acc[0, d + 10] == 1   # (10, y, theta=0) -> D + 10
    assert acc[90, d + 7] == 1   # (x, 7, theta=90) -> D + 7


def test_vote_conservation(oracle):
    for n_theta in (1, 7, 180, 720):
        c, s = synth.q15_table(n_theta)
        b = synth.random_image(n_theta, 50, 40, "binary")
        e = oracle.compact(b)
        acc = oracle.hough_accumulate(e, 50, 40, c, s)
        assert int(acc.sum()) == len(e) * n_theta
        assert (acc.sum(axis=1) == len(e)).all()


@pytest.mark.parametrize("n_theta", [180, 720, 1024])
def test_lines_closed_forms(oracle, n_theta):
    g = load_golden("hough_pins.json")
    c, s = synth.q15_table(n_theta)
    w, h = 400, 300
    d = oracle.rho_offset(w, h)
    # horizontal line of N pixels at y0: acc[n/2][D + y0] = N = max(acc)
    y0, n = 123, w
    e = np.array([(y0 << 16) | x for x in range(n)], np.uint32)
    acc = oracle.hough_accumulate(e, w, h, c, s)
    assert acc[n_theta // 2, d + y0] == n and acc.max() == n
    # vertical line at x0: acc[0][D + x0] = N
    x0 = 77
    e = np.array([(y << 16) | x0 for y in range(h)], np.uint32)
    acc = oracle.hough_accumulate(e, w, h, c, s)
    assert acc[0, d + x0] == h and acc.max() == h
    # x + y = 200 at theta = 45 deg; x - y = 100 at theta = 135 deg
    dg = g["diagonal_x_plus_y"]
    e = np.array([((dg["c"] - x) << 16) | x for x in range(dg["c"] + 1)], np.uint32)
    acc = oracle.hough_accumulate(e, w, h, c, s)
    assert acc[n_theta // 4, d + dg["rho_minus_D"]] == dg["c"] + 1
    ad = g["antidiagonal_x_minus_y"]
    e = np.array([(y << 16) | (y + ad["c"]) for y in range(h) if y + ad["c"] < w], np.uint32)
    acc = oracle.hough_accumulate(e, w, h, c, s)
    assert acc[3 * n_theta // 4, d + ad["rho_minus_D"]] == len(e)


def test_exhaustive_4x4_subsets_additivity(oracle):
    # Brute force: all 2^16 subsets of a 4x4 patch at an offset; each accumulator
    # equals the sum of its pixels' single-pixel accumulators (pinned above).
    c, s = synth.q15_table(8)
    w, h, ox, oy = 16, 16, 5, 9
    pix = [((oy + i // 4) << 16) | (ox + i % 4) for i in range(16)]
    singles = np.stack([oracle.hough_accumulate(np.array([p], np.uint32), w, h, c, s).ravel()
                        for p in pix]).astype(np.int64)
    masks = ((np.arange(1 << 16)[:, None] >> np.arange(16)[None, :]) & 1).astype(np.int64)
    want = masks @ singles
    for m in range(1 << 16):
        e = np.array([pix[i] for i in range(16) if (m >> i) & 1], np.uint32)
        acc = oracle.hough_accumulate(e, w, h, c, s)
        assert np.array_equal(acc.ravel(), want[m])


def test_range_error_on_oversized_table(oracle):
    c = np.array([65536], np.int32)   # |C| > 2^15 pushes rho out of [0, n_rho)
    s = np.array([0], np.int32)
    with pytest.raises(oracle.OracleError):
        oracle.hough_accumulate(np.array([(0 << 16) | 9], np.uint32), 10, 1, c, s)


# ----------------------------------------------------------------------------
# Peaks (DESIGN R13, R14)
# ----------------------------------------------------------------------------
def _brute_peaks(acc, ht, hr, min_votes, k):
    n_t, n_r = acc.shape
    cands = []
    for t in range(n_t):
        for r in range(n_r):
            v = int(acc[t, r])
            if v < max(1, min_votes):
                continue
            win = [(int(acc[tt, rr]), -tt, -rr)
                   for tt in range(max(0, t - ht), min(n_t, t + ht + 1))
                   for rr in range(max(0, r - hr), min(n_r, r + hr + 1))]
            if max(win) == (v, -t, -r):
                cands.append((v, -t, -r))
    cands.sort(reverse=True)
    out = [(-tt, -rr, v) for v, tt, rr in cands[:k]]
    return out + [(-1, -1, 0)] * (k - len(out)), min(k, len(cands))


def _as_tuples(peaks):
    return [(int(p["theta_bin"]), int(p["rho_bin"]), int(p["votes"])) for p in peaks]


def test_peaks_brute_force_random(oracle):
    rng = np.random.default_rng(3)
    for trial in range(60):
        n_t, n_r = int(rng.integers(1, 12)), int(rng.integers(1, 30))
        acc = rng.integers(0, int(rng.integers(1, 6)), size=(n_t, n_r)).astype(np.uint32)
        ht, hr = int(rng.integers(0, 4)), int(rng.integers(0, 6))
        mv, k = int(rng.integers(0, 4)), int(rng.integers(1, 9))
        got, n = oracle.hough_peaks(acc, ht, hr, mv, k)
        want, wn = _brute_peaks(acc, ht, hr, mv, k)
        assert n == wn and _as_tuples(got) == want, (trial, acc, ht, hr, mv, k)


def test_peaks_window_zero_is_sort(oracle):
    rng = np.random.default_rng(4)
    acc = rng.integers(0, 4, size=(6, 9)).astype(np.uint32)
    got, n = oracle.hough_peaks(acc, 0, 0, 1, 100)
    t, r = np.nonzero(acc)
    order = sorted(zip(acc[t, r].tolist(), (-t).tolist(), (-r).tolist()), reverse=True)
    assert n == len(order)
    assert _as_tuples(got)[:n] == [(-a, -b, v) for v, a, b in order]


def test_peaks_special_cases(oracle):
    acc = np.zeros((10, 20), np.uint32)
    got, n = oracle.hough_peaks(acc, 2, 3, 1, 4)
    assert n == 0 and _as_tuples(got) == [(-1, -1, 0)] * 4          # all-zero
    acc[4, 7] = 9
    got, n = oracle.hough_peaks(acc, 2, 3, 1, 4)
    assert n == 1 and _as_tuples(got)[0] == (4, 7, 9)
    acc[8, 15] = 9   # equal maxima farther apart than the window -> lower theta first
    got, n = oracle.hough_peaks(acc, 2, 3, 1, 4)
    assert n == 2 and _as_tuples(got)[:2] == [(4, 7, 9), (8, 15, 9)]
    acc[5, 8] = 9    # tie inside the window: the lower (theta, rho) wins
    got, n = oracle.hough_peaks(acc, 2, 3, 1, 4)
    assert _as_tuples(got)[:2] == [(4, 7, 9), (8, 15, 9)] and n == 2
    got, n = oracle.hough_peaks(acc, 2, 3, 10, 4)                   # min_votes
    assert n == 0


def test_peaks_no_theta_wraparound(oracle):
    acc = np.zeros((10, 5), np.uint32)
    acc[0, 2] = 5
    acc[9, 2] = 7
    got, n = oracle.hough_peaks(acc, 2, 1, 1, 4)
    assert n == 2 and _as_tuples(got)[:2] == [(9, 2, 7), (0, 2, 5)]


# ----------------------------------------------------------------------------
# End to end: planted lanes (S:527 generalised; BASELINE.json configs[0])
# ----------------------------------------------------------------------------
def test_cfg1_planted_lanes_recovered(oracle):
    cfg = synth.CONFIGS["cfg1"]
    img = synth.gen_frame("cfg1", 0)
    c, s = synth.q15_table(cfg.n_theta)
    r = oracle.detect(img, cfg.threshold, c, s, cfg.half_theta, cfg.half_rho,
                      cfg.min_votes, cfg.k)
    d = oracle.rho_offset(cfg.width, cfg.height)
    assert r["n_peaks"] == 2
    found = sorted((int(p["theta_bin"]), int(p["rho_bin"]) - d) for p in r["peaks"])
    lanes = sorted((l["theta_deg"], l["r"]) for l in
                   load_golden("hough_pins.json")["cfg1_lanes"]["lanes"])
    for (t, rho), (th, rr) in zip(found, lanes):
        assert abs(t - th) <= 1.0 and abs(rho - rr) <= 3.5, (found, lanes)
    assert int(r["acc"].sum()) == r["n_edges"] * cfg.n_theta
    assert np.array_equal(r["binary"], oracle.sobel_binarize(img, cfg.threshold))


def test_detect_composes_stages(oracle):
    img = synth.gen_frame("cfg1", 0)
    c, s = synth.q15_table(180)
    r = oracle.detect(img, 200, c, s, 2, 8, 1, 5)
    b = oracle.sobel_binarize(img, 200)
    e = oracle.compact(b)
    acc = oracle.hough_accumulate(e, 320, 240, c, s)
    pk, n = oracle.hough_peaks(acc, 2, 8, 1, 5)
    assert np.array_equal(r["edges"], e) and np.array_equal(r["acc"], acc)
    assert _as_tuples(r["peaks"]) == _as_tuples(pk) and r["n_peaks"] == n


# ----------------------------------------------------------------------------
# NEXT 3: lanes module (DESIGN R26-R28)
# ----------------------------------------------------------------------------
def test_lanes_golden_spec_examples(oracle):
    g = load_golden("lanes_pins.json")
    c, s = synth.q15_table(180)
    for case in g["peak_to_line"]:
        d = oracle.rho_offset(case["w"], case["h"])
        got = oracle.peak_to_line((case["theta_bin"], d + case["rho"], 1), case["w"], case["h"],
                                  c, s)
        assert got == tuple(case["segment"]), case["cite"]
    for case in g["extract_segments"]:
        b = np.zeros((case["h"], case["w"]), np.uint8)
        for a, e in case["white"]:
            b[case["row"], a:e] = 255
        d = oracle.rho_offset(case["w"], case["h"])
        segs, n = oracle.extract_segments(b, (90, d + case["row"], 1), c, s, case["fill_gap"],
                                          case["min_len"])
        assert segs == [tuple(x) for x in case["segments"]] and n == len(segs), case["cite"]
    for case in g["find_peaks"]:
        acc = np.zeros((case["n_theta"], case["n_rho"]), np.uint32)
        for t, r, v in case["cells"]:
            acc[t, r] = v
        pk, n = oracle.hough_peaks_nms(acc, case["nhood"][0], case["nhood"][1], 1, 0, 1, case["k"])
        assert [tuple(int(v) for v in p) for p in pk[:n]] == [tuple(x) for x in case["peaks"]]


def test_nms_greedy_differs_from_window_maxima(oracle):
    # hand chain along rho (half_rho = 2): 5 @ r0, 6 @ r2, 7 @ r4.  The window
    # maxima are {r4}; greedy picks r4, suppresses r2..r6, and r0 (5) is then
    # the largest unsuppressed cell -- a pick that is not a window maximum.
    acc = np.zeros((1, 12), np.uint32)
    acc[0, [0, 2, 4]] = [5, 6, 7]
    pk, n = oracle.hough_peaks_nms(acc, 0, 2, 1, 0, 1, 4)
    assert n == 2 and [tuple(int(v) for v in p) for p in pk[:2]] == [(0, 4, 7), (0, 0, 5)]
    wp, wn = oracle.hough_peaks(acc, 0, 2, 1, 4)
    assert wn == 1 and tuple(int(v) for v in wp[0]) == (0, 4, 7)


def test_nms_ratio_threshold_is_inclusive(oracle):
    acc = np.zeros((5, 40), np.uint32)
    acc[0, 0], acc[2, 20], acc[4, 39] = 10, 5, 4
    pk, n = oracle.hough_peaks_nms(acc, 0, 0, 1, 1, 2, 8)  # votes >= 0.5 * 10
    assert n == 2 and [int(p["votes"]) for p in pk[:2]] == [10, 5]
    pk, n = oracle.hough_peaks_nms(acc, 0, 0, 6, 0, 1, 8)  # min_votes floor
    assert n == 1
    pk, n = oracle.hough_peaks_nms(np.zeros((3, 3), np.uint32), 1, 1, 1, 0, 1, 2)
    assert n == 0 and all(tuple(int(v) for v in p) == (-1, -1, 0) for p in pk)


def test_nms_sparse_far_cells_is_a_sort(oracle):
    # cells pairwise farther apart than the window: greedy = all cells by key
    rng = np.random.default_rng(3)
    for trial in range(20):
        acc = np.zeros((60, 200), np.uint32)
        cells = []
        for t in range(0, 60, 7):
            for r in range(0, 200, 19):
                if rng.random() < 0.5:
                    v = int(rng.integers(1, 6))
                    acc[t, r] = v
                    cells.append((v, -t, -r))
        cells.sort(reverse=True)
        want = [(-t, -r, v) for v, t, r in cells][:12]
        pk, n = oracle.hough_peaks_nms(acc, 3, 9, 1, 0, 1, 12)
        assert [tuple(int(v) for v in p) for p in pk[:n]] == want


def test_nms_first_pick_is_global_max_and_picks_are_separated(oracle):
    rng = np.random.default_rng(4)
    for trial in range(30):
        acc = rng.integers(0, 9, size=(int(rng.integers(1, 30)), int(rng.integers(1, 60)))).astype(np.uint32)
        ht, hr, k = int(rng.integers(0, 4)), int(rng.integers(0, 8)), int(rng.integers(1, 10))
        pk, n = oracle.hough_peaks_nms(acc, ht, hr, 1, 0, 1, k)
        wp, wn = oracle.hough_peaks(acc, ht, hr, 1, 1)
        if acc.max() == 0:
            assert n == 0
            continue
        assert tuple(int(v) for v in pk[0]) == tuple(int(v) for v in wp[0])  # the key maximum
        picks = [tuple(int(v) for v in p) for p in pk[:n]]
        for i in range(n):
            for j in range(i):  # a later pick is outside every earlier window
                assert abs(picks[i][0] - picks[j][0]) > ht or abs(picks[i][1] - picks[j][1]) > hr
            assert picks[i][2] == acc[picks[i][0], picks[i][1]]
        assert [p[2] for p in picks] == sorted((p[2] for p in picks), reverse=True)
        # maximality: every unpicked positive cell is inside some pick's window
        if n < k:
            for t, r in zip(*np.nonzero(acc)):
                assert any(abs(t - p[0]) <= ht and abs(r - p[1]) <= hr for p in picks)


def test_peak_to_line_endpoints_on_line_and_border(oracle):
    # every returned end is the rounding of a point of the rectangle's border
    # that lies on x cos + y sin = rho, so it is within 0.5*sqrt(2) px of the
    # line (in the table's own cos/sin) and at the border (up to rounding)
    rng = np.random.default_rng(5)
    for n_theta in (180, 720):
        c, s = synth.q15_table(n_theta)
        for trial in range(200):
            w, h = int(rng.integers(2, 700)), int(rng.integers(2, 500))
            d = oracle.rho_offset(w, h)
            t = int(rng.integers(0, n_theta))
            r = int(rng.integers(-d, d + 1))
            seg = oracle.peak_to_line((t, d + r, 1), w, h, c, s)
            cc, ss = c[t] / 32768.0, s[t] / 32768.0
            if seg is None:
                # a miss: every corner is strictly on one side of the line
                vals = [x * cc + y * ss - r for x in (0, w - 1) for y in (0, h - 1)]
                assert all(v > 0 for v in vals) or all(v < 0 for v in vals)
                continue
            for x, y in ((seg[0], seg[1]), (seg[2], seg[3])):
                assert 0 <= x <= w - 1 and 0 <= y <= h - 1
                assert abs(x * cc + y * ss - r) <= 0.5 * (abs(cc) + abs(ss)) + 1e-9
                assert min(x, y, w - 1 - x, h - 1 - y) <= 0  # on the border
            assert (seg[0], seg[1]) <= (seg[2], seg[3])


def test_extract_segments_gap_rule_and_vertical_walk(oracle):
    c, s = synth.q15_table(180)
    d = oracle.rho_offset(120, 90)
    b = np.zeros((90, 120), np.uint8)
    # column x = 30 (theta bin 0 walks along y): runs 0..29 and 56..89 (gap 26)
    b[0:30, 30] = 255
    b[56:90, 30] = 255
    segs, n = oracle.extract_segments(b, (0, d + 30, 1), c, s, 25, 20)
    assert segs == [(30, 0, 30, 29), (30, 56, 30, 89)]
    segs, n = oracle.extract_segments(b, (0, d + 30, 1), c, s, 26, 20)  # gap 26 <= 26
    assert segs == [(30, 0, 30, 89)]
    segs, n = oracle.extract_segments(b, (0, d + 30, 1), c, s, 25, 33)  # second run is 33 long
    assert segs == [(30, 56, 30, 89)]
    # capacity: count reported, list truncated
    b2 = np.zeros((10, 200), np.uint8)
    b2[4, ::3] = 255
    segs, n = oracle.extract_segments(b2, (90, oracle.rho_offset(200, 10) + 4, 1), c, s, 0, 0,
                                      cap=5)
    assert n == 67 and len(segs) == 5 and segs[0] == (0, 4, 0, 4)


# ----------------------------------------------------------------------------
# NEXT 4: SPEC float64 trig mode (DESIGN R29)
# ----------------------------------------------------------------------------
def test_f64_table_spec_pins():
    c, s = synth.f64_table(180)
    assert c[0] == 1.0 and s[0] == 0.0 and c[90] == 0.0 and s[90] == 1.0
    assert s[179] == s[1] and c[179] == -c[1]                            # S:200, Eq. 4
    assert np.all(np.abs(c * c + s * s - 1.0) <= 1e-12)
    for n in (2, 8, 720, 1024):
        c, s = synth.f64_table(n)
        for k in range(1, n // 2):
            assert s[n - k] == s[k] and c[n - k] == -c[k]


def test_f64_rho_of_and_accumulate_spec_examples(oracle):
    c, s = synth.f64_table(180)
    w, h = 64, 48
    d = oracle.rho_offset(w, h)

    def rho_bins(x, y):
        acc = oracle.hough_accumulate_f64(np.array([(y << 16) | x], np.uint32), w, h, c, s)
        return [int(np.nonzero(acc[t])[0][0]) for t in range(180)]

    assert all(r == d for r in rho_bins(0, 0))                 # S:229 origin
    assert rho_bins(10, 33)[0] == d + 10                       # S:230 r = x at theta 0
    assert rho_bins(21, 7)[90] == d + 7                        # S:231 r = y at 90 degrees
    row = np.array([(5 << 16) | x for x in (3, 4, 5)], np.uint32)
    acc = oracle.hough_accumulate_f64(row, w, h, c, s)
    assert acc[90, d + 5] == 3 and acc.sum() == 3 * 180
    assert oracle.hough_accumulate_f64(np.zeros(0, np.uint32), w, h, c, s).sum() == 0


def test_f64_matches_exact_rational_away_from_ties(oracle):
    # exact r = x*c + y*s over the rationals of the double table entries; the
    # double evaluation may only differ where r + 1/2 is within 1e-9 of an integer
    c, s = synth.f64_table(180)
    rng = np.random.default_rng(41)
    w, h = 1280, 720
    d = oracle.rho_offset(w, h)
    xs, ys = rng.integers(0, w, 300), rng.integers(0, h, 300)
    e = ((ys.astype(np.uint32) << 16) | xs.astype(np.uint32))
    for i in range(len(e)):
        acc = oracle.hough_accumulate_f64(e[i:i + 1], w, h, c, s)
        got = acc.argmax(axis=1) - d
        for t in range(0, 180, 7):
            r = Fraction(int(xs[i])) * Fraction(float(c[t])) + Fraction(int(ys[i])) * Fraction(float(s[t]))
            want = math.floor(r + Fraction(1, 2))
            near = abs((r + Fraction(1, 2)) - round(r + Fraction(1, 2))) < Fraction(1, 10 ** 9)
            assert got[t] == want or near, (i, t)


def test_f64_within_one_bin_of_q15_and_conservation(oracle):
    cf, sf = synth.f64_table(180)
    cq, sq = synth.q15_table(180)
    rng = np.random.default_rng(42)
    w, h = 320, 240
    e = ((rng.integers(0, h, 2000).astype(np.uint32) << 16) |
         rng.integers(0, w, 2000).astype(np.uint32))
    af = oracle.hough_accumulate_f64(e, w, h, cf, sf)
    aq = oracle.hough_accumulate(e, w, h, cq, sq)
    assert af.sum() == aq.sum() == len(e) * 180
    for i in range(0, 2000, 97):
        bf = oracle.hough_accumulate_f64(e[i:i + 1], w, h, cf, sf).argmax(axis=1)
        bq = oracle.hough_accumulate(e[i:i + 1], w, h, cq, sq).argmax(axis=1)
        assert np.abs(bf.astype(int) - bq.astype(int)).max() <= 1
