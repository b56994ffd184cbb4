"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit-exact.

Everything here is integer work, so the bar is exact equality of the binary
map, the edge count, the edge list as a set (DESIGN R15), the accumulator and
the peaks (DESIGN R22).  Inputs are the seeded generators of
paper_2212_09460_b200.synth; expected values come only from oracle/.
"""
import numpy as np
import pytest

from paper_2212_09460_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ld():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2212_09460_b200 import build, ld as _ld
    build.build()
    return _ld


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def peak_tuples(p, n=None):
    p = np.asarray(p).reshape(-1, 3)
    out = [(int(a), int(b), int(np.uint32(np.int32(c)))) for a, b, c in p]
    return out


def oracle_peak_tuples(pk):
    return [(int(p["theta_bin"]), int(p["rho_bin"]), int(p["votes"])) for p in pk]


def gpu_sobel(ld, frames, threshold, pitch_pad=0):
    """frames: uint8 [B][H][W] numpy -> binary, sorted edge lists, counts."""
    b, h, w = frames.shape
    pitch = ld._round_up(w, 16) + pitch_pad
    buf = np.zeros((b, h, pitch), np.uint8)
    buf[:, :, :w] = frames
    g = cuda(buf)
    img = ld.make_image(w, h, pitch, h * pitch, b)
    stride = ld._round_up(max(h * max(w - 2, 0), 1), 4)
    binary = torch.full((b, h, pitch), 7, dtype=torch.uint8, device="cuda")
    edges = torch.full((b, stride), -1, dtype=torch.int32, device="cuda")
    counts = torch.full((b,), -1, dtype=torch.int32, device="cuda")
    ld.ld_sobel_binarize(g, img, threshold, binary, edges, stride, counts)
    torch.cuda.synchronize()
    cnt = counts.cpu().numpy()
    el = edges.cpu().numpy().view(np.uint32)
    lists = [np.sort(el[i, :cnt[i]]) for i in range(b)]
    return binary.cpu().numpy()[:, :, :w], lists, cnt


# ----------------------------------------------------------------------------
# Stage 1-2: Sobel + binarize + compaction
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg4"])
def test_sobel_configs(ld, oracle, name):
    cfg = synth.CONFIGS[name]
    img = synth.gen_frame(name, 0)
    binary, lists, cnt = gpu_sobel(ld, img[None], cfg.threshold)
    want = oracle.sobel_binarize(img, cfg.threshold)
    assert np.array_equal(binary[0], want)
    we = oracle.compact(want)
    assert cnt[0] == len(we)
    assert np.array_equal(lists[0], np.sort(we))


def test_sobel_cfg5_full_size(ld, oracle):
    img = synth.gen_frame("cfg5", 0)
    binary, lists, cnt = gpu_sobel(ld, img[None], 200)
    want = oracle.sobel_binarize(img, 200)
    assert np.array_equal(binary[0], want)
    assert np.array_equal(lists[0], np.sort(oracle.compact(want)))


def test_sobel_batch_cfg3_frames(ld, oracle):
    frames = synth.gen_batch("cfg3", 0, 6)
    binary, lists, cnt = gpu_sobel(ld, frames, 200)
    for i in range(6):
        want = oracle.sobel_binarize(frames[i], 200)
        assert np.array_equal(binary[i], want), i
        assert np.array_equal(lists[i], np.sort(oracle.compact(want))), i


SIZES = [(1, 1), (1, 5), (2, 2), (3, 3), (4, 3), (17, 2), (2, 40), (5, 7), (15, 16), (16, 16),
         (17, 17), (31, 33), (223, 65), (224, 64), (225, 66), (241, 129), (256, 300), (300, 1)]


@pytest.mark.parametrize("w,h", SIZES)
@pytest.mark.parametrize("kind", ["uniform", "binary"])
def test_sobel_fuzz_sizes(ld, oracle, w, h, kind):
    img = synth.random_image(w * 1000 + h, w, h, kind)
    for t in (0, 1, 199, 200, 201, 1530, 1531, -5):
        binary, lists, cnt = gpu_sobel(ld, img[None], t, pitch_pad=16 if w % 2 else 0)
        want = oracle.sobel_binarize(img, t)
        assert np.array_equal(binary[0], want), (w, h, t)
        assert np.array_equal(lists[0], np.sort(oracle.compact(want))), (w, h, t)


def test_sobel_bands_match_whole(ld, oracle):
    # row bands with a 1-row halo (ld_image.row_begin/row_end) == whole frame
    img = synth.random_image(77, 200, 150, "uniform")
    want = oracle.sobel_binarize(img, 300)
    pitch = 208
    full = np.zeros((150, pitch), np.uint8)
    full[:, :200] = img
    got_rows, got_edges = [], []
    for rb, re in [(0, 1), (1, 37), (37, 64), (64, 65), (65, 149), (149, 150)]:
        r0, r1 = max(rb - 1, 0), min(re + 1, 150)
        g = cuda(full[r0:r1].copy())
        im = ld.make_image(200, 150, pitch, (r1 - r0) * pitch, 1, rb, re)
        stride = ld._round_up((re - rb) * 198, 4)
        b = torch.zeros((re - rb, pitch), dtype=torch.uint8, device="cuda")
        e = torch.zeros((max(stride, 4),), dtype=torch.int32, device="cuda")
        c = torch.zeros((1,), dtype=torch.int32, device="cuda")
        ld.ld_sobel_binarize(g, im, 300, b, e, stride, c)
        torch.cuda.synchronize()
        got_rows.append(b.cpu().numpy()[:, :200])
        got_edges.append(e.cpu().numpy().view(np.uint32)[: int(c.item())])
    assert np.array_equal(np.concatenate(got_rows), want)
    assert np.array_equal(np.sort(np.concatenate(got_edges)), np.sort(oracle.compact(want)))


# ----------------------------------------------------------------------------
# Stage 3: voting
# ----------------------------------------------------------------------------
def gpu_vote_list(ld, edge_lists, w, h, n_theta, flags=0):
    c, s = synth.q15_table(n_theta)
    b = len(edge_lists)
    stride = ld._round_up(max(max(len(e) for e in edge_lists), 1), 4)
    el = np.zeros((b, stride), np.uint32)
    for i, e in enumerate(edge_lists):
        el[i, :len(e)] = e
    counts = cuda(np.array([len(e) for e in edge_lists], np.int32))
    acc = ld.hough_accumulate(cuda(el.view(np.int32)), counts, stride, w, h, c, s, flags=flags)
    torch.cuda.synchronize()
    return acc.cpu().numpy().view(np.uint32)


# LD_VOTE_PLAIN forces the plain kernel; without it a symmetric table (every
# synth.q15_table) selects the half-angle paired kernel (NEXT 2)
VOTE_MODES = ["paired", "plain"]


@pytest.fixture(params=VOTE_MODES)
def vote_mode(request):
    """ld_hough_accumulate_opt flags of the mode."""
    from paper_2212_09460_b200 import ld as _ld
    return _ld.LD_VOTE_PLAIN if request.param == "plain" else 0


@pytest.mark.parametrize("n_theta", [1, 2, 3, 4, 5, 180, 181, 720, 1024, 2048])
def test_vote_random_lists(ld, oracle, n_theta, vote_mode):
    c, s = synth.q15_table(n_theta)
    rng = np.random.default_rng(n_theta)
    w, h = 301, 203
    lists = []
    for n in (0, 1, 5, 4099):
        xs, ys = rng.integers(0, w, n), rng.integers(0, h, n)
        lists.append(((ys.astype(np.uint32) << 16) | xs.astype(np.uint32)))
    got = gpu_vote_list(ld, lists, w, h, n_theta, vote_mode)
    for i, e in enumerate(lists):
        assert np.array_equal(got[i], oracle.hough_accumulate(e, w, h, c, s)), (n_theta, len(e))


def test_vote_extreme_corners_and_tiny(ld, oracle, vote_mode):
    for w, h in [(1, 1), (2, 1), (16384, 1), (1, 16384), (16384, 16384)]:
        c, s = synth.q15_table(64)
        corners = sorted({(0, 0), (w - 1, 0), (0, h - 1), (w - 1, h - 1)})
        e = np.array([(y << 16) | x for x, y in corners], np.uint32)
        got = gpu_vote_list(ld, [e], w, h, 64, vote_mode)
        assert np.array_equal(got[0], oracle.hough_accumulate(e, w, h, c, s)), (w, h)


def test_vote_collinear_hotspot(ld, oracle, vote_mode):
    # thousands of votes into the same bin (same-address atomics)
    c, s = synth.q15_table(180)
    e = np.array([(100 << 16) | x for x in range(1000)] * 3, np.uint32)
    got = gpu_vote_list(ld, [e], 1000, 200, 180, vote_mode)
    want = oracle.hough_accumulate(e, 1000, 200, c, s)
    assert np.array_equal(got[0], want) and want.max() == 3000


def test_vote_asymmetric_table_uses_plain_path(ld, oracle):
    # one entry off the symmetry C[n-t] = -C[t]: the paired kernel would be
    # wrong for that row, so the host must fall back (results stay exact)
    c, s = synth.q15_table(180)
    c = c.copy()
    c[30] += 1
    rng = np.random.default_rng(5)
    w, h = 640, 360
    xs, ys = rng.integers(0, w, 20000), rng.integers(0, h, 20000)
    e = (ys.astype(np.uint32) << 16) | xs.astype(np.uint32)
    counts = cuda(np.array([len(e)], np.int32))
    acc = ld.hough_accumulate(cuda(e.view(np.int32)[None]), counts, len(e), w, h, c, s)
    torch.cuda.synchronize()
    assert np.array_equal(acc.cpu().numpy().view(np.uint32)[0],
                          oracle.hough_accumulate(e, w, h, c, s))


def test_vote_paired_equals_plain_on_frames(ld):
    cfg = synth.CONFIGS["cfg3"]
    c, s = synth.q15_table(cfg.n_theta)
    _, edges, counts, stride = ld.sobel_binarize(cuda(synth.gen_batch("cfg3", 0, 4)), cfg.threshold,
                                                 want_binary=False)
    a1, h1 = ld.hough_accumulate(edges, counts, stride, 1280, 720, c, s, want_hint=True)
    a0, h0 = ld.hough_accumulate(edges, counts, stride, 1280, 720, c, s, want_hint=True,
                                 flags=ld.LD_VOTE_PLAIN)
    assert torch.equal(a0, a1)
    # both kernels' chunk maxima (the sparse peak search's input, R30) are
    # exact or the "examine" marker
    check_chunk_maxima(a0, h0)
    check_chunk_maxima(a1, h1)
    p0, n0 = ld.hough_peaks(a0, cfg.half_theta, cfg.half_rho, 1, cfg.k, hint=h0)
    p1, n1 = ld.hough_peaks(a1, cfg.half_theta, cfg.half_rho, 1, cfg.k, hint=h1)
    assert torch.equal(p0, p1) and torch.equal(n0, n1)


def check_chunk_maxima(acc, hint):
    """The hint's chunk maxima (DESIGN R30): chunk q of frame f covers the
    1 KB-aligned bytes [(c0 + q) * 1024, +1024) of the accumulator, c0 = frame
    start // 1024; its entry is exactly the maximum of the frame's counters in
    it (chunks shared by voting blocks or frames included)."""
    b, nt, nr = acc.shape
    ncells = nt * nr
    n_seg = (ncells * 4 + 1023) // 1024 + 1
    seg = hint[-b * n_seg * 4:].view(torch.int32).cpu().numpy().view(np.uint32).reshape(b, n_seg)
    A = acc.cpu().numpy().view(np.uint32).reshape(b, ncells)
    base = acc.data_ptr()
    for f in range(b):
        start = base + f * ncells * 4
        c0 = start // 1024
        first = (start - c0 * 1024) // 4  # counters of chunk 0 before the frame
        padded = np.zeros(n_seg * 256, np.uint32)
        padded[first:first + ncells] = A[f]
        true = padded.reshape(n_seg, 256).max(axis=1)
        used = (start + ncells * 4 - 1) // 1024 - c0 + 1
        s_ = seg[f, :used]
        ok = s_ == true[:used]
        assert ok.all(), (f, np.flatnonzero(~ok)[:5], s_[~ok][:5], true[:used][~ok][:5])


def test_vote_range_error(ld):
    c = np.array([40000], np.int32)
    s = np.array([0], np.int32)
    with pytest.raises(ld.LdError) as ei:
        gpu_vote_list_raw(ld, c, s)
    assert ei.value.status == ld.LD_ERR_RANGE


def gpu_vote_list_raw(ld, c, s):
    el = torch.zeros((4,), dtype=torch.int32, device="cuda")
    cnt = torch.zeros((1,), dtype=torch.int32, device="cuda")
    acc = torch.zeros((1, len(c), 2 * ld.ld_rho_offset(10, 10) + 1), dtype=torch.int32,
                      device="cuda")
    ld.ld_hough_accumulate(el, cnt, 4, 1, 10, 10, len(c), c, s, acc)


# ----------------------------------------------------------------------------
# Stage 4: peaks
# ----------------------------------------------------------------------------
# ld_hough_peaks_opt flags forcing each search kernel
PEAK_KERNEL_FLAGS = {"auto": 0, "stream": 2, "tile": 4, "band": 8}

def test_peaks_random_small(ld, oracle):
    rng = np.random.default_rng(9)
    for trial in range(40):
        b = int(rng.integers(1, 4))
        n_t, n_r = int(rng.integers(1, 40)), int(rng.integers(1, 700))
        acc = rng.integers(0, int(rng.integers(1, 8)), size=(b, n_t, n_r)).astype(np.uint32)
        ht, hr = int(rng.integers(0, 5)), int(rng.integers(0, 30))
        mv, k = int(rng.integers(0, 5)), int(rng.choice([1, 2, 4, 7, 64, 1024]))
        peaks, npk = ld.hough_peaks(cuda(acc.view(np.int32)), ht, hr, mv, k)
        torch.cuda.synchronize()
        peaks, npk = peaks.cpu().numpy(), npk.cpu().numpy()
        for f in range(b):
            want, wn = oracle.hough_peaks(acc[f], ht, hr, mv, k)
            assert npk[f] == wn, (trial, f)
            assert peak_tuples(peaks[f]) == oracle_peak_tuples(want), (trial, f)


def test_peaks_window_zero_many_candidates(ld, oracle):
    # every nonzero cell is a candidate: exercises the candidate buffer merges
    rng = np.random.default_rng(2)
    acc = rng.integers(0, 1000, size=(1, 37, 1999)).astype(np.uint32)
    for k in (1, 5, 1024):
        peaks, npk = ld.hough_peaks(cuda(acc.view(np.int32)), 0, 0, 1, k)
        want, wn = oracle.hough_peaks(acc[0], 0, 0, 1, k)
        assert int(npk[0]) == wn and peak_tuples(peaks[0].cpu()) == oracle_peak_tuples(want)


# ----------------------------------------------------------------------------
# End to end (ld_detect_batch) on every config
# ----------------------------------------------------------------------------
def run_detect(ld, name, frames):
    cfg = synth.CONFIGS[name]
    c, s = synth.q15_table(cfg.n_theta)
    b, h, w = frames.shape
    det = ld.Detector(w, h, b, cfg.n_theta, c, s, cfg.threshold, cfg.k, cfg.half_theta,
                      cfg.half_rho, cfg.min_votes, export_acc=True)
    g = torch.zeros((b, h, det.pitch), dtype=torch.uint8, device="cuda")
    g[:, :, :w] = cuda(frames)
    peaks, npk, counts, acc = det(g)
    torch.cuda.synchronize()
    return det, peaks, npk, counts, acc


def check_frame(oracle, name, frame, peaks_f, npk_f, count_f, acc_f):
    cfg = synth.CONFIGS[name]
    c, s = synth.q15_table(cfg.n_theta)
    r = oracle.detect(frame, cfg.threshold, c, s, cfg.half_theta, cfg.half_rho, cfg.min_votes,
                      cfg.k)
    assert int(count_f) == r["n_edges"]
    if acc_f is not None:
        assert np.array_equal(acc_f, r["acc"])
    assert int(npk_f) == r["n_peaks"]
    assert peak_tuples(peaks_f) == oracle_peak_tuples(r["peaks"])


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg5"])
def test_detect_single_frame_configs(ld, oracle, name):
    frames = synth.gen_frame(name, 0)[None]
    det, peaks, npk, counts, acc = run_detect(ld, name, frames)
    check_frame(oracle, name, frames[0], peaks.cpu().numpy()[0], npk.cpu()[0], counts.cpu()[0],
                acc.cpu().numpy().view(np.uint32)[0])


def test_detect_cfg4_two_frames(ld, oracle):
    frames = synth.gen_batch("cfg4", 0, 2)
    det, peaks, npk, counts, acc = run_detect(ld, "cfg4", frames)
    for i in range(2):
        check_frame(oracle, "cfg4", frames[i], peaks.cpu().numpy()[i], npk.cpu()[i],
                    counts.cpu()[i], acc[i].cpu().numpy().view(np.uint32))


def test_detect_cfg3_full_batch_sampled(ld, oracle):
    # full BASELINE size and launch configuration (256 frames); sampled frames
    # against the oracle, invariants on every frame
    cfg = synth.CONFIGS["cfg3"]
    frames = synth.gen_batch("cfg3")
    det, peaks, npk, counts, acc = run_detect(ld, "cfg3", frames)
    sums = acc.view(256, -1).sum(dim=1, dtype=torch.int64).cpu().numpy()
    cnt = counts.cpu().numpy().astype(np.int64)
    assert np.array_equal(sums, cnt * cfg.n_theta)   # vote conservation, every frame
    pk = peaks.cpu().numpy()
    for i in (0, 1, 77, 128, 254, 255):
        check_frame(oracle, "cfg3", frames[i], pk[i], npk.cpu()[i], cnt[i],
                    acc[i].cpu().numpy().view(np.uint32))


def test_detect_deterministic(ld):
    frames = synth.gen_batch("cfg3", 0, 16)
    a = run_detect(ld, "cfg3", frames)
    b = run_detect(ld, "cfg3", frames)
    for x, y in zip(a[1:], b[1:]):
        assert torch.equal(x, y)


def test_detect_host_path_matches_device(ld):
    cfg = synth.CONFIGS["cfg3"]
    c, s = synth.q15_table(cfg.n_theta)
    frames = synth.gen_batch("cfg3", 0, 20)
    _, peaks, npk, counts, _ = run_detect(ld, "cfg3", frames)
    hd = ld.HostDetector(1280, 720, 20, cfg.n_theta, c, s, cfg.threshold, cfg.k, cfg.half_theta,
                         cfg.half_rho, cfg.min_votes, chunk_frames=6)
    host = torch.from_numpy(frames).pin_memory()
    hp, hn, hc = hd(host)
    assert torch.equal(hp, peaks.cpu()) and torch.equal(hn, npk.cpu())
    assert torch.equal(hc, counts.cpu())


def test_banded_accumulators_sum_to_whole(ld, oracle):
    # cfg5 split in row bands: per-band accumulators summed == whole == oracle
    cfg = synth.CONFIGS["cfg5"]
    c, s = synth.q15_table(cfg.n_theta)
    img = synth.gen_frame("cfg5", 0)
    W = H = 4096
    want = oracle.hough_accumulate(oracle.compact(oracle.sobel_binarize(img, 200)), W, H, c, s)
    g_all = cuda(img)
    for n in (2, 8):
        total = None
        for r in range(n):
            rb, re = r * H // n, (r + 1) * H // n
            r0, r1 = max(rb - 1, 0), min(re + 1, H)
            im = ld.make_image(W, H, W, (r1 - r0) * W, 1, rb, re)
            stride = ld._round_up((re - rb) * (W - 2), 4)
            e = torch.empty((stride,), dtype=torch.int32, device="cuda")
            cnt = torch.empty((1,), dtype=torch.int32, device="cuda")
            ld.ld_sobel_binarize(g_all[r0:r1], im, 200, None, e, stride, cnt)
            acc = ld.hough_accumulate(e, cnt, stride, W, H, c, s)
            total = acc if total is None else total + acc
        torch.cuda.synchronize()
        assert np.array_equal(total.cpu().numpy().view(np.uint32)[0], want), n


@pytest.mark.parametrize("kernel", ["auto", "stream", "tile", "band"])
def test_peaks_all_kernels_windows(ld, oracle, kernel):
    # the default choice (warp-strip kernel for narrow windows, else the CTA
    # streaming kernel), the forced CTA streaming kernel, the tiled kernel and
    # the generic band kernel all agree with the oracle
    flags = PEAK_KERNEL_FLAGS[kernel]
    rng = np.random.default_rng(31)
    for trial, (ht, hr) in enumerate([(0, 0), (0, 5), (1, 1), (2, 29), (7, 44), (10, 116),
                                      (12, 3), (13, 2), (3, 240), (20, 300)]):
        acc = rng.integers(0, 6, size=(2, 61, 1201)).astype(np.uint32)
        acc[1, 30, 600] = 50      # one dominant peak
        peaks, npk = ld.hough_peaks(cuda(acc.view(np.int32)), ht, hr, 1, 16, flags=flags)
        torch.cuda.synchronize()
        for f in range(2):
            want, wn = oracle.hough_peaks(acc[f], ht, hr, 1, 16)
            assert int(npk[f]) == wn, (kernel, ht, hr, f)
            assert peak_tuples(peaks[f].cpu()) == oracle_peak_tuples(want), (kernel, ht, hr, f)


def test_peaks_many_tiles_merge(ld, oracle):
    # cfg5-like geometry: thousands of tile lists merged per frame
    rng = np.random.default_rng(5)
    acc = rng.integers(0, 30, size=(1, 1024, 2001)).astype(np.uint32)
    peaks, npk = ld.hough_peaks(cuda(acc.view(np.int32)), 10, 116, 1, 64)
    want, wn = oracle.hough_peaks(acc[0], 10, 116, 1, 64)
    assert int(npk[0]) == wn and peak_tuples(peaks[0].cpu()) == oracle_peak_tuples(want)


def test_banded_detector_ranks_emulated(ld, oracle):
    # dist.BandedDetector for every rank of world N in one process (no process
    # group: its allreduce is then the identity), partial accumulators summed
    # here == whole-image oracle; world 1 gives the oracle's peaks directly
    from paper_2212_09460_b200 import dist as pdist
    cfg = synth.CONFIGS["cfg5"]
    c, s = synth.q15_table(cfg.n_theta)
    img = synth.gen_frame("cfg5", 0)
    W = H = 4096
    r = oracle.detect(img, cfg.threshold, c, s, cfg.half_theta, cfg.half_rho, cfg.min_votes,
                      cfg.k)
    for world in (1, 3, 8):
        total = None
        for rank in range(world):
            det = pdist.BandedDetector(W, H, cfg.n_theta, c, s, cfg.threshold, cfg.k,
                                       cfg.half_theta, cfg.half_rho, cfg.min_votes, rank, world)
            det.load(img)
            peaks, npk, acc, cnt = det()
            part = acc.clone()
            total = part if total is None else total + part
        torch.cuda.synchronize()
        assert np.array_equal(total.cpu().numpy().view(np.uint32)[0], r["acc"]), world
        if world == 1:
            assert int(cnt[0]) == r["n_edges"]
            assert int(npk[0]) == r["n_peaks"]
            assert peak_tuples(peaks[0].cpu()) == oracle_peak_tuples(r["peaks"])


def test_banded_detector_more_ranks_than_rows(ld, oracle):
    from paper_2212_09460_b200 import dist as pdist
    img = synth.random_image(3, 50, 5, "uniform")
    c, s = synth.q15_table(180)
    want = oracle.hough_accumulate(oracle.compact(oracle.sobel_binarize(img, 200)), 50, 5, c, s)
    total = None
    for rank in range(8):
        det = pdist.BandedDetector(50, 5, 180, c, s, 200, 4, 2, 8, 1, rank, 8)
        det.load(img)
        _, _, acc, _ = det()
        total = acc.clone() if total is None else total + acc
    torch.cuda.synchronize()
    assert np.array_equal(total.cpu().numpy().view(np.uint32)[0], want)


@pytest.mark.parametrize("kernel", ["auto", "stream", "band"])
def test_peaks_ties_and_plateaus(ld, oracle, kernel):
    # equal maxima inside one window (plateaus, equal values left/right/above/
    # below) exercise the exact (theta, rho) tie-break; small value range makes
    # ties everywhere
    flags = PEAK_KERNEL_FLAGS[kernel]
    rng = np.random.default_rng(77)
    for trial, (ht, hr, k) in enumerate([(2, 29, 4), (1, 3, 64), (0, 0, 1024), (7, 44, 8),
                                         (10, 116, 64), (12, 5, 16), (3, 0, 32), (3, 4, 64),
                                         (0, 64, 2), (2, 15, 64), (1, 14, 7)]):
        acc = rng.integers(0, 3, size=(3, 97, 1500)).astype(np.uint32)
        acc[0, 40:43, 700:705] = 9                    # plateau
        acc[1, 10, 100] = acc[1, 10, 103] = acc[1, 12, 101] = 7
        acc[2, :, 1499] = 5                           # column of equal values at the edge
        peaks, npk = ld.hough_peaks(cuda(acc.view(np.int32)), ht, hr, 1, k, flags=flags)
        torch.cuda.synchronize()
        for f in range(3):
            want, wn = oracle.hough_peaks(acc[f], ht, hr, 1, k)
            assert int(npk[f]) == wn, (kernel, trial, f)
            assert peak_tuples(peaks[f].cpu()) == oracle_peak_tuples(want), (kernel, trial, f)


def test_peaks_stream_theta_chunks_single_frame(ld, oracle):
    # one frame -> the streaming kernel splits theta into chunks with a
    # half_theta-row halo; peaks near chunk seams must match
    rng = np.random.default_rng(8)
    acc = rng.integers(0, 40, size=(1, 1024, 3001)).astype(np.uint32)
    for t in (0, 15, 16, 17, 31, 32, 33, 63, 64, 500, 1023):
        acc[0, t, (t * 37) % 3001] = 1000 + t
    for ht, hr, k in [(10, 116, 64), (2, 29, 4), (0, 0, 16), (12, 300, 32)]:
        peaks, npk = ld.hough_peaks(cuda(acc.view(np.int32)), ht, hr, 1, k)
        want, wn = oracle.hough_peaks(acc[0], ht, hr, 1, k)
        assert int(npk[0]) == wn and peak_tuples(peaks[0].cpu()) == oracle_peak_tuples(want)


# ----------------------------------------------------------------------------
# NEXT 4: paper-literal zero-padded border and SPEC 8-bit clamp (DESIGN R23, R24)
# ----------------------------------------------------------------------------
def gpu_sobel_ex(ld, frames, threshold, flags, pitch_pad=0):
    b, h, w = frames.shape
    pitch = ld._round_up(w, 16) + pitch_pad
    buf = np.zeros((b, h, pitch), np.uint8)
    buf[:, :, :w] = frames
    g = cuda(buf)
    img = ld.make_image(w, h, pitch, h * pitch, b)
    stride = ld._round_up(max(h * w, 1), 4)
    binary = torch.full((b, h, pitch), 7, dtype=torch.uint8, device="cuda")
    edges = torch.full((b, stride), -1, dtype=torch.int32, device="cuda")
    counts = torch.full((b,), -1, dtype=torch.int32, device="cuda")
    ld.ld_sobel_binarize_ex(g, img, threshold, flags, binary, edges, stride, counts)
    torch.cuda.synchronize()
    cnt = counts.cpu().numpy()
    el = edges.cpu().numpy().view(np.uint32)
    return binary.cpu().numpy()[:, :, :w], [np.sort(el[i, :cnt[i]]) for i in range(b)], cnt


@pytest.mark.parametrize("flags", [1, 2, 3])
@pytest.mark.parametrize("w,h", [(1, 1), (2, 3), (5, 7), (16, 16), (17, 17), (223, 65),
                                 (225, 66), (256, 300), (300, 1)])
def test_sobel_flags_fuzz(ld, oracle, flags, w, h):
    img = synth.random_image(w * 7 + h, w, h, "uniform")
    for t in (-1, 0, 1, 200, 255, 256, 1530, 1531):
        binary, lists, cnt = gpu_sobel_ex(ld, img[None], t, flags, pitch_pad=16 if w % 3 else 0)
        want = oracle.sobel_binarize_ex(img, t, flags)
        assert np.array_equal(binary[0], want), (w, h, t, flags)
        assert np.array_equal(lists[0], np.sort(oracle.compact(want))), (w, h, t, flags)


def test_sobel_zero_pad_bands_match_whole(ld, oracle):
    # row bands (1-row halo) in zero-padded mode == the whole frame: halo rows
    # inside the image are real rows, only rows -1 and H are padding
    img = synth.random_image(91, 200, 150, "uniform")
    want = oracle.sobel_binarize_ex(img, 300, oracle.ZERO_PAD)
    pitch = 208
    full = np.zeros((150, pitch), np.uint8)
    full[:, :200] = img
    rows, edges = [], []
    for rb, re in [(0, 1), (1, 37), (37, 64), (64, 149), (149, 150)]:
        r0, r1 = max(rb - 1, 0), min(re + 1, 150)
        g = cuda(full[r0:r1].copy())
        im = ld.make_image(200, 150, pitch, (r1 - r0) * pitch, 1, rb, re)
        stride = ld._round_up((re - rb) * 200, 4)
        b = torch.zeros((re - rb, pitch), dtype=torch.uint8, device="cuda")
        e = torch.zeros((stride,), dtype=torch.int32, device="cuda")
        c = torch.zeros((1,), dtype=torch.int32, device="cuda")
        ld.ld_sobel_binarize_ex(g, im, 300, ld.LD_FLAG_ZERO_PAD, b, e, stride, c)
        torch.cuda.synchronize()
        rows.append(b.cpu().numpy()[:, :200])
        edges.append(e.cpu().numpy().view(np.uint32)[: int(c.item())])
    assert np.array_equal(np.concatenate(rows), want)
    assert np.array_equal(np.sort(np.concatenate(edges)), np.sort(oracle.compact(want)))


def test_sobel_flags_reject_unknown_bits_and_short_stride(ld):
    g = torch.zeros((4, 16), dtype=torch.uint8, device="cuda")
    img = ld.make_image(10, 4, 16, 64, 1)
    c = torch.zeros((1,), dtype=torch.int32, device="cuda")
    e = torch.zeros((64,), dtype=torch.int32, device="cuda")
    with pytest.raises(ld.LdError):
        ld.ld_sobel_binarize_ex(g, img, 10, 4, None, e, 64, c)
    with pytest.raises(ld.LdError):  # zero-pad needs rows * width = 40 > 32
        ld.ld_sobel_binarize_ex(g, img, 10, ld.LD_FLAG_ZERO_PAD, None, e, 32, c)
    ld.ld_sobel_binarize_ex(g, img, 10, 0, None, e, 32, c)  # 4 * 8 = 32 is enough


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_detect_zero_pad_end_to_end(ld, oracle, name):
    cfg = synth.CONFIGS[name]
    c, s = synth.q15_table(cfg.n_theta)
    frame = synth.gen_frame(name, 0)
    h, w = frame.shape
    det = ld.Detector(w, h, 1, cfg.n_theta, c, s, cfg.threshold, cfg.k, cfg.half_theta,
                      cfg.half_rho, cfg.min_votes, export_acc=True, flags=ld.LD_FLAG_ZERO_PAD)
    g = torch.zeros((1, h, det.pitch), dtype=torch.uint8, device="cuda")
    g[:, :, :w] = cuda(frame[None])
    peaks, npk, counts, acc = det(g)
    torch.cuda.synchronize()
    b = oracle.sobel_binarize_ex(frame, cfg.threshold, oracle.ZERO_PAD)
    e = oracle.compact(b)
    want_acc = oracle.hough_accumulate(e, w, h, c, s)
    want_pk, want_n = oracle.hough_peaks(want_acc, cfg.half_theta, cfg.half_rho, cfg.min_votes,
                                         cfg.k)
    assert int(counts[0]) == len(e)
    assert np.array_equal(acc[0].cpu().numpy().view(np.uint32), want_acc)
    assert int(npk[0]) == want_n
    assert peak_tuples(peaks[0].cpu()) == oracle_peak_tuples(want_pk)


# ----------------------------------------------------------------------------
# NEXT 1: theta slices of an accumulator (ld_hough_peaks_ex) and theta-sharded
# detection (dist.ThetaShardedDetector)
# ----------------------------------------------------------------------------
def oracle_all_candidates(oracle, big, ht, hr, mv):
    allp, n = oracle.hough_peaks(big, ht, hr, mv, big.size)
    return [(int(p["theta_bin"]), int(p["rho_bin"]), int(p["votes"])) for p in allp[:n]]


def oracle_slice_peaks(cands, t0, t1, k):
    # the definition restricted to candidate rows [t0, t1) of the full accumulator
    return [c for c in cands if t0 <= c[0] < t1][:k]


@pytest.mark.parametrize("kernel", ["auto", "stream", "band"])
def test_peaks_ex_theta_slices(ld, oracle, kernel):
    flags = PEAK_KERNEL_FLAGS[kernel]
    rng = np.random.default_rng(123)
    for trial, (nt, ht, hr, k) in enumerate([(180, 2, 29, 4), (1024, 10, 116, 64),
                                              (97, 3, 5, 16), (60, 0, 0, 8), (33, 7, 44, 8)]):
        big = rng.integers(0, 12 if trial % 2 else 5000, size=(nt, 1201)).astype(np.uint32)
        cands = oracle_all_candidates(oracle, big, ht, hr, 1)
        for (t0, t1) in [(0, nt), (0, nt // 3), (nt // 3, 2 * nt // 3), (2 * nt // 3, nt),
                         (nt // 2, nt // 2), (nt - 1, nt)]:
            g0, g1 = max(t0 - ht, 0), min(t1 + ht, nt)
            # an empty shard with no halo still passes a 1-row accumulator
            # (the ABI requires n_theta >= 1); its candidate range is empty
            sl = np.ascontiguousarray(big[g0:max(g1, g0 + 1)])[None]
            peaks, npk = ld.hough_peaks(cuda(sl.view(np.int32)), ht, hr, 1, k,
                                        cand_rows=(t0 - g0, t1 - g0), theta_offset=g0,
                                        flags=flags)
            torch.cuda.synchronize()
            want = oracle_slice_peaks(cands, t0, t1, k)
            assert int(npk[0]) == len(want), (kernel, trial, t0, t1)
            got = peak_tuples(peaks[0].cpu())[:len(want)]
            assert got == want, (kernel, trial, t0, t1)


@pytest.mark.parametrize("keys_rows", ["slice", "all"])
def test_peaks_ex_theta_slices_hint_from_acc(ld, oracle, keys_rows):
    """ld_hough_hint_from_acc on theta slices (halo rows included), with its
    keys taken from the candidate rows only or from every row (the search
    must drop the others), through the fused search with candidate rows and a
    theta offset: the definition restricted to those rows (oracle)."""
    rng = np.random.default_rng(321)
    W, H = 360, 480  # 2 ld_rho_offset + 1 = 1201 bins: sizes the hint buffer
    for trial, (nt, ht, hr, k) in enumerate([(180, 2, 29, 4), (1024, 10, 116, 64),
                                              (97, 3, 5, 16), (33, 7, 44, 8)]):
        big = rng.integers(0, 12 if trial % 2 else 5000, size=(nt, 1201)).astype(np.uint32)
        # a few strong peaks, so that the hint certifies a bound
        for j in range(3 * k):
            big[rng.integers(0, nt), rng.integers(0, 1201)] = 20000 + j
        cands = oracle_all_candidates(oracle, big, ht, hr, 1)
        for (t0, t1) in [(0, nt), (0, nt // 3), (nt // 3, 2 * nt // 3), (2 * nt // 3, nt)]:
            g0, g1 = max(t0 - ht, 0), min(t1 + ht, nt)
            sl = cuda(np.ascontiguousarray(big[g0:g1])[None].view(np.int32))
            rows = (t0 - g0, t1 - g0)
            hint = ld.hint_from_acc(sl, W, H, cand_rows=rows if keys_rows == "slice" else None)
            peaks, npk = ld.hough_peaks(sl, ht, hr, 1, k, cand_rows=rows, theta_offset=g0,
                                        hint=hint)
            torch.cuda.synchronize()
            want = oracle_slice_peaks(cands, t0, t1, k)
            assert int(npk[0]) == len(want), (trial, t0, t1)
            assert peak_tuples(peaks[0].cpu())[:len(want)] == want, (trial, t0, t1)


@pytest.mark.parametrize("name,nf", [("cfg2", 1), ("cfg3", 6), ("cfg4", 2)])
def test_hint_from_acc_whole_frames(ld, oracle, name, nf):
    """The hint of a finished accumulator (what a row-band all_reduce sum
    needs) gives the exact peaks, and describes the chunks exactly."""
    cfg = synth.CONFIGS[name]
    c, s = synth.q15_table(cfg.n_theta)
    frames = synth.gen_batch(name, 0, nf) if cfg.batch > 1 else synth.gen_frame(name, 0)[None]
    b, h, w = frames.shape
    _, edges, counts, stride = ld.sobel_binarize(cuda(frames), cfg.threshold, want_binary=False)
    acc = ld.hough_accumulate(edges, counts, stride, w, h, c, s)
    hint = ld.hint_from_acc(acc, w, h)
    check_chunk_maxima(acc, hint)
    p0, n0 = ld.hough_peaks(acc, cfg.half_theta, cfg.half_rho, cfg.min_votes, cfg.k)
    p1, n1 = ld.hough_peaks(acc, cfg.half_theta, cfg.half_rho, cfg.min_votes, cfg.k, hint=hint)
    _, nt, nr = acc.shape
    wsb = ld.ld_hough_peaks_workspace_bytes(b, nt, nr, cfg.k)
    ws = torch.zeros((wsb,), dtype=torch.uint8, device="cuda")
    p2 = torch.empty((b, cfg.k, 3), dtype=torch.int32, device="cuda")
    n2 = torch.empty((b,), dtype=torch.int32, device="cuda")
    ld.ld_hough_peaks_hinted(acc, b, nt, nr, cfg.half_theta, cfg.half_rho, cfg.min_votes, cfg.k,
                             hint, hint.numel(), p2, n2, ws, wsb)
    torch.cuda.synchronize()
    assert torch.equal(p0, p1) and torch.equal(n0, n1)
    assert torch.equal(p0, p2) and torch.equal(n0, n2)
    # the search was resolved by the hint (the sparse path ran)
    head = (4 * b + 255) // 256 * 256
    assert ws[head:head + 4 * b].view(torch.int32).min().item() == 1
    A = acc.cpu().numpy().view(np.uint32)
    for f in range(b):
        pk, npk = oracle.hough_peaks(A[f], cfg.half_theta, cfg.half_rho, cfg.min_votes, cfg.k)
        assert int(n1.cpu()[f]) == npk
        assert peak_tuples(p1.cpu().numpy()[f]) == oracle_peak_tuples(pk)


def test_theta_sharded_detector_emulated(ld, oracle):
    # every rank of world N in one process: the whole-image edge list stands in
    # for the all-gathered band lists; per-rank top-k lists merged on device
    from paper_2212_09460_b200 import dist as pdist
    cfg = synth.CONFIGS["cfg5"]
    c, s = synth.q15_table(cfg.n_theta)
    img = synth.gen_frame("cfg5", 0)
    W = H = 4096
    r = oracle.detect(img, cfg.threshold, c, s, cfg.half_theta, cfg.half_rho, cfg.min_votes,
                      cfg.k, want_binary=False, want_acc=False)
    _, edges, counts, stride = ld.sobel_binarize(cuda(img[None]), cfg.threshold, want_binary=False)
    assert int(counts[0]) == r["n_edges"]
    for world in (1, 2, 3, 8):
        allp, alln = [], []
        for rank in range(world):
            det = pdist.ThetaShardedDetector(W, H, cfg.n_theta, c, s, cfg.threshold, cfg.k,
                                             cfg.half_theta, cfg.half_rho, cfg.min_votes,
                                             rank, world)
            det.vote_and_peaks(edges[0], counts, stride)
            allp.append(det.peaks[0].clone())
            alln.append(det.n_peaks.clone())
        p, n = pdist.merge_peak_lists(torch.stack(allp), torch.cat(alln), det.n_rho, cfg.k)
        torch.cuda.synchronize()
        assert int(n[0]) == r["n_peaks"], world
        assert peak_tuples(p.cpu()) == oracle_peak_tuples(r["peaks"]), world


# ----------------------------------------------------------------------------
# Peak hint (DESIGN R25): ld_hough_accumulate_hint votes identically, and
# ld_hough_peaks_hinted returns exactly ld_hough_peaks' result; the per-frame
# threshold left in the workspace never exceeds the frame's k-th best
# candidate value (the property that makes the hint safe).
# ----------------------------------------------------------------------------
def _hint_case(ld, oracle, frames, cfg, kernel=None, monkeypatch=None, check_oracle=True):
    c, s = synth.q15_table(cfg.n_theta)
    g = cuda(frames)
    _, edges, counts, stride = ld.sobel_binarize(g, cfg.threshold, want_binary=False)
    b, h, w = frames.shape
    acc0 = ld.hough_accumulate(edges, counts, stride, w, h, c, s)
    acc, hint = ld.hough_accumulate(edges, counts, stride, w, h, c, s, want_hint=True)
    assert torch.equal(acc0, acc)
    check_chunk_maxima(acc, hint)
    p0, n0 = ld.hough_peaks(acc, cfg.half_theta, cfg.half_rho, cfg.min_votes, cfg.k)
    # a copy of the accumulator at another address: the chunk maxima do not
    # describe it, so the search falls back to dense -- same peaks
    pc, nc = ld.hough_peaks(acc.clone(), cfg.half_theta, cfg.half_rho, cfg.min_votes, cfg.k,
                            hint=hint)
    assert torch.equal(p0, pc) and torch.equal(n0, nc)
    _, nt, nr = acc.shape
    wsb = ld.ld_hough_peaks_workspace_bytes(b, nt, nr, cfg.k)
    ws = torch.zeros((wsb,), dtype=torch.uint8, device="cuda")
    p1 = torch.empty((b, cfg.k, 3), dtype=torch.int32, device="cuda")
    n1 = torch.empty((b,), dtype=torch.int32, device="cuda")
    ld.ld_hough_peaks_hinted(acc, b, nt, nr, cfg.half_theta, cfg.half_rho, cfg.min_votes, cfg.k,
                             hint, hint.numel(), p1, n1, ws, wsb)
    torch.cuda.synchronize()
    assert torch.equal(n0, n1) and torch.equal(p0, p1)
    gtau = ws[:4 * b].view(torch.int32).cpu().numpy().view(np.uint32)
    # the hinted search without the sparse stage (R30) gives the same peaks
    p2, n2 = ld.hough_peaks(acc, cfg.half_theta, cfg.half_rho, cfg.min_votes, cfg.k, hint=hint,
                            flags=ld.LD_PEAKS_DENSE)
    assert torch.equal(n0, n2) and torch.equal(p0, p2)
    n1c, p1c = n1.cpu().numpy(), p1.cpu().numpy()
    for f in range(b):
        if n1c[f] == cfg.k:
            assert gtau[f] <= np.uint32(np.int32(p1c[f, cfg.k - 1, 2])), (f, gtau[f])
    if check_oracle:
        A = acc.cpu().numpy().view(np.uint32)
        for f in range(b):
            pk, npk = oracle.hough_peaks(A[f], cfg.half_theta, cfg.half_rho, cfg.min_votes, cfg.k)
            assert int(n1c[f]) == npk
            assert peak_tuples(p1c[f]) == oracle_peak_tuples(pk)  # sentinels included
    return gtau, p1c, n1c


# (frame counts cover every launch shape of the fused search: clusters of 8
# CTAs per frame (1-18 frames), 4 (19-37), 2 (38-73, cfg4's 64), one 1024-
# thread CTA (74-147) and one 512-thread CTA (>= 148: cfg3's 256, in
# test_gpu_full_configs))
@pytest.mark.parametrize("name,nf", [("cfg1", 1), ("cfg2", 1), ("cfg3", 6), ("cfg3", 24),
                                     ("cfg3", 100), ("cfg4", 2), ("cfg5", 1)])
def test_hinted_peaks_identical(ld, oracle, name, nf):
    cfg = synth.CONFIGS[name]
    frames = synth.gen_batch(name, 0, nf) if cfg.batch > 1 else synth.gen_frame(name, 0)[None]
    gtau, p, n = _hint_case(ld, oracle, frames, cfg)
    # the hint is not vacuous on the road configs: the start threshold reached
    # a real candidate value for some frame
    if name in ("cfg2", "cfg3"):
        assert gtau.max() > 1


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("k", [1, 4, 64])
def test_hinted_peaks_ties_and_sparse(ld, oracle, seed, k):
    # low-contrast frames (many equal small counts: ties everywhere) and a few
    # hard lines; several window sizes through the warp and stream kernels
    rng = np.random.default_rng(100 + seed)
    frames = rng.integers(0, 2, size=(3, 96, 160), dtype=np.uint8) * 255
    frames[1] = 0
    frames[1, 40:43, :] = 255
    frames[2, :, 70:72] = 255
    for (ht, hr) in [(0, 4), (2, 29), (3, 64), (7, 44), (10, 116)]:
        cfg = synth.Config("t", 160, 96, 3, 200, 90, k, ht, hr)
        _hint_case(ld, oracle, frames, cfg)


@pytest.mark.parametrize("k", [64, 256, 1024])
def test_hinted_peaks_large_k(ld, oracle, k):
    # k past the best 32 m keys the fused search selects first (the full-sort
    # continuation), and past what the hint can certify (dense fallback), on
    # road frames with min_votes 1 (thousands of local maxima)
    cfg = synth.CONFIGS["cfg3"]
    frames = synth.gen_batch("cfg3", 3, 2)
    cfg = synth.Config("k%d" % k, 1280, 720, 2, cfg.threshold, cfg.n_theta, k, cfg.half_theta,
                       cfg.half_rho)
    _hint_case(ld, oracle, frames, cfg)


@pytest.mark.parametrize("min_votes", [150, 200, 260, 100000])
def test_hinted_peaks_min_votes_floor(ld, oracle, min_votes):
    # a floor at, above or far above the k-th best peak (fewer than k
    # candidates, or none): the keys below the floor end the verification, the
    # result is the oracle's (sentinels included)
    cfg = synth.CONFIGS["cfg2"]
    frames = np.stack([synth.gen_frame("cfg2", 0), synth.gen_batch("cfg3", 5, 1)[0]])
    cfg = synth.Config("mv", 1280, 720, 2, cfg.threshold, cfg.n_theta, cfg.k, cfg.half_theta,
                       cfg.half_rho, min_votes)
    _hint_case(ld, oracle, frames, cfg)


def test_hint_of_another_accumulator(ld, oracle):
    # a hint recorded while voting frame A, used with frame B's accumulator
    # of the same shape at another address: the header matches, the chunk
    # maxima are not used (other address) and A's keys are verified against
    # B's counts (a key must hold its value there) -- B's exact peaks
    cfg = synth.CONFIGS["cfg2"]
    c, s = synth.q15_table(cfg.n_theta)
    fa = synth.gen_frame("cfg2", 0)[None]
    fb = synth.gen_batch("cfg3", 11, 1)
    _, ea, ca, sa = ld.sobel_binarize(cuda(fa), cfg.threshold, want_binary=False)
    _, eb, cb, sb = ld.sobel_binarize(cuda(fb), cfg.threshold, want_binary=False)
    _, hint_a = ld.hough_accumulate(ea, ca, sa, 1280, 720, c, s, want_hint=True)
    acc_b = ld.hough_accumulate(eb, cb, sb, 1280, 720, c, s)
    p1, n1 = ld.hough_peaks(acc_b, cfg.half_theta, cfg.half_rho, cfg.min_votes, cfg.k, hint=hint_a)
    p0, n0 = ld.hough_peaks(acc_b, cfg.half_theta, cfg.half_rho, cfg.min_votes, cfg.k)
    torch.cuda.synchronize()
    assert torch.equal(p0, p1) and torch.equal(n0, n1)
    A = acc_b.cpu().numpy().view(np.uint32)
    pk, npk = oracle.hough_peaks(A[0], cfg.half_theta, cfg.half_rho, cfg.min_votes, cfg.k)
    assert int(n1.cpu()[0]) == npk
    assert peak_tuples(p1.cpu().numpy()[0]) == oracle_peak_tuples(pk)


def test_hint_header_mismatch_ignored(ld, oracle):
    cfg = synth.CONFIGS["cfg2"]
    frames = synth.gen_frame("cfg2", 0)[None]
    c, s = synth.q15_table(cfg.n_theta)
    _, edges, counts, stride = ld.sobel_binarize(cuda(frames), cfg.threshold, want_binary=False)
    acc, hint = ld.hough_accumulate(edges, counts, stride, 1280, 720, c, s, want_hint=True)
    p0, n0 = ld.hough_peaks(acc, cfg.half_theta, cfg.half_rho, 1, cfg.k)
    bad = hint.clone()
    bad[:4] = 0  # wrong magic: ignored
    p1, n1 = ld.hough_peaks(acc, cfg.half_theta, cfg.half_rho, 1, cfg.k, hint=bad)
    assert torch.equal(p0, p1) and torch.equal(n0, n1)
    with pytest.raises(ld.LdError):  # too small a hint buffer
        ld.ld_hough_accumulate_hint(edges, counts, stride, 1, 1280, 720, cfg.n_theta, c, s, acc,
                                    hint, 64)


_MISALIGNED_CACHE = {}


@pytest.mark.parametrize("shift", [1, 2, 3])
@pytest.mark.parametrize("name", ["cfg1", "cfg4"])
def test_hinted_peaks_misaligned_accumulator(ld, oracle, name, shift):
    # an accumulator that starts 4/8/12 bytes past a 16-byte boundary (the
    # ABI asks only for 4-byte alignment): the window tests read 16-byte
    # vectors aligned to the allocation, so frame edges fall inside vectors;
    # voting and the hinted search against the oracle, frame by frame
    cfg = synth.CONFIGS[name]
    nf = 2
    frames = synth.gen_batch(name, 0, nf) if cfg.batch > 1 else np.stack(
        [synth.gen_frame(name, 0)] * nf)
    c, s = synth.q15_table(cfg.n_theta)
    b, h, w = frames.shape
    _, edges, counts, stride = ld.sobel_binarize(cuda(frames), cfg.threshold, want_binary=False)
    nr = 2 * ld.ld_rho_offset(w, h) + 1
    buf = torch.full((b * cfg.n_theta * nr + 4,), -1, dtype=torch.int32, device="cuda")
    acc = buf[shift:shift + b * cfg.n_theta * nr].view(b, cfg.n_theta, nr)
    hb = ld.ld_hough_hint_bytes(b, w, h, cfg.n_theta)
    hint = torch.empty((hb,), dtype=torch.uint8, device="cuda")
    ld.ld_hough_accumulate_hint(edges, counts, stride, b, w, h, cfg.n_theta, c, s, acc, hint, hb)
    wsb = ld.ld_hough_peaks_workspace_bytes(b, cfg.n_theta, nr, cfg.k)
    ws = torch.zeros((wsb,), dtype=torch.uint8, device="cuda")
    pk = torch.empty((b, cfg.k, 3), dtype=torch.int32, device="cuda")
    npk = torch.empty((b,), dtype=torch.int32, device="cuda")
    ld.ld_hough_peaks_hinted(acc, b, cfg.n_theta, nr, cfg.half_theta, cfg.half_rho,
                             cfg.min_votes, cfg.k, hint, hb, pk, npk, ws, wsb)
    torch.cuda.synchronize()
    assert buf[:shift].eq(-1).all() and buf[shift + acc.numel():].eq(-1).all()
    A = acc.cpu().numpy().view(np.uint32)
    pkc, npc = pk.cpu().numpy(), npk.cpu().numpy()
    for f in range(b):
        key = (name, f)
        if key not in _MISALIGNED_CACHE:  # the oracle's result does not depend on the shift
            want = oracle.hough_accumulate(
                oracle.compact(oracle.sobel_binarize(frames[f], cfg.threshold)), w, h, c, s)
            _MISALIGNED_CACHE[key] = (want, oracle.hough_peaks(want, cfg.half_theta,
                                                               cfg.half_rho, cfg.min_votes,
                                                               cfg.k))
        want, (opk, onp) = _MISALIGNED_CACHE[key]
        assert np.array_equal(A[f], want)
        assert int(npc[f]) == onp
        assert peak_tuples(pkc[f]) == oracle_peak_tuples(opk)


# ----------------------------------------------------------------------------
# Lanes module (NEXT 3, DESIGN R26-R28): greedy NMS, peak_to_line,
# extract_segments against the oracle
# ----------------------------------------------------------------------------
def _np_peaks(p, n):
    return [tuple(int(v) for v in q) for q in np.asarray(p)[:n]]


@pytest.mark.parametrize("ratio", [(0, 1), (1, 2), (3, 4), (5, 4)])
def test_nms_random_accumulators(ld, oracle, ratio):
    rng = np.random.default_rng(31)
    for trial in range(12):
        b = int(rng.integers(1, 4))
        nt, nr = int(rng.integers(1, 50)), int(rng.integers(1, 400))
        acc = rng.integers(0, int(rng.integers(1, 12)), size=(b, nt, nr)).astype(np.uint32)
        ht, hr = int(rng.integers(0, 4)), int(rng.integers(0, 20))
        mv, k = int(rng.integers(0, 4)), int(rng.choice([1, 2, 4, 9]))
        pk, npk = ld.hough_peaks_nms(cuda(acc.view(np.int32)), ht, hr, mv, k, ratio=ratio)
        torch.cuda.synchronize()
        pk, npk = pk.cpu().numpy(), npk.cpu().numpy()
        for f in range(b):
            want, wn = oracle.hough_peaks_nms(acc[f], ht, hr, mv, ratio[0], ratio[1], k)
            assert npk[f] == wn, (trial, f)
            assert peak_tuples(pk[f]) == oracle_peak_tuples(want), (trial, f)


def test_nms_on_detected_frames(ld, oracle):
    cfg = synth.CONFIGS["cfg3"]
    c, s = synth.q15_table(cfg.n_theta)
    frames = synth.gen_batch("cfg3", 0, 3)
    _, edges, counts, stride = ld.sobel_binarize(cuda(frames), cfg.threshold, want_binary=False)
    acc = ld.hough_accumulate(edges, counts, stride, 1280, 720, c, s)
    pk, npk = ld.hough_peaks_nms(acc, 5, 40, 1, 8, ratio=(1, 2))
    torch.cuda.synchronize()
    A = acc.cpu().numpy().view(np.uint32)
    for f in range(3):
        want, wn = oracle.hough_peaks_nms(A[f], 5, 40, 1, 1, 2, 8)
        assert int(npk[f]) == wn and peak_tuples(pk[f].cpu()) == oracle_peak_tuples(want)


def test_peak_lines_match_oracle(ld, oracle):
    rng = np.random.default_rng(32)
    for n_theta in (180, 720, 1024):
        c, s = synth.q15_table(n_theta)
        for (w, h) in [(512, 512), (1280, 720), (37, 900), (2, 2)]:
            d = oracle.rho_offset(w, h)
            k = 64
            pk = np.zeros((1, k, 3), np.int32)
            pk[0, :, 0] = rng.integers(0, n_theta, k)
            pk[0, :, 1] = rng.integers(0, 2 * d + 1, k)
            pk[0, :, 2] = 1
            pk[0, :4, 0] = [0, n_theta // 2, n_theta // 4, 0]  # the axis-aligned and 45-degree cases
            pk[0, :4, 1] = [d + 100 % max(w, 1), d + 3, d, d]
            npk = np.array([k - 3], np.int32)  # the last 3 slots are not peaks
            lines, hit = ld.peak_lines(cuda(pk), cuda(npk), w, h, c, s)
            torch.cuda.synchronize()
            lines, hit = lines.cpu().numpy(), hit.cpu().numpy()
            for i in range(k):
                want = oracle.peak_to_line(tuple(pk[0, i]), w, h, c, s) if i < k - 3 else None
                assert (hit[0, i] == 1) == (want is not None), (n_theta, w, h, i)
                if want is not None:
                    assert tuple(int(v) for v in lines[0, i]) == want, (n_theta, w, h, i)


def test_extract_segments_match_oracle(ld, oracle):
    cfg = synth.CONFIGS["cfg3"]
    c, s = synth.q15_table(cfg.n_theta)
    frames = synth.gen_batch("cfg3", 0, 2)
    binary, edges, counts, stride = ld.sobel_binarize(cuda(frames), cfg.threshold)
    acc = ld.hough_accumulate(edges, counts, stride, 1280, 720, c, s)
    pk, npk = ld.hough_peaks(acc, cfg.half_theta, cfg.half_rho, 1, 16)
    bpitch = binary.contiguous()
    for fill_gap, min_len in [(20, 40), (0, 0), (5, 100)]:
        segs, nseg = ld.extract_segments(bpitch, pk, npk, c, s, fill_gap, min_len,
                                         max_segments=32)
        torch.cuda.synchronize()
        segs, nseg = segs.cpu().numpy(), nseg.cpu().numpy()
        B = bpitch.cpu().numpy()
        P, N = pk.cpu().numpy(), npk.cpu().numpy()
        for f in range(2):
            for i in range(16):
                if i >= N[f]:
                    assert nseg[f, i] == 0
                    continue
                want, wn = oracle.extract_segments(B[f], tuple(P[f, i]), c, s, fill_gap, min_len,
                                                   cap=32)
                assert nseg[f, i] == wn, (fill_gap, min_len, f, i)
                got = [tuple(int(v) for v in segs[f, i, j]) for j in range(min(wn, 32))]
                assert got == want, (fill_gap, min_len, f, i)


def test_extract_segments_vertical_and_synthetic(ld, oracle):
    c, s = synth.q15_table(180)
    b = np.zeros((1, 90, 128), np.uint8)
    b[0, 0:30, 30] = 255
    b[0, 56:90, 30] = 255
    b[0, 45, :] = 255
    b[0, 45, 60:75] = 0
    d = oracle.rho_offset(128, 90)
    pk = np.array([[[0, d + 30, 1], [90, d + 45, 1], [45, d + 50, 1]]], np.int32)
    npk = np.array([3], np.int32)
    for fg, ml in [(25, 20), (26, 20), (14, 10), (15, 0)]:
        segs, nseg = ld.extract_segments(cuda(b), cuda(pk), cuda(npk), c, s, fg, ml, 8)
        torch.cuda.synchronize()
        segs, nseg = segs.cpu().numpy(), nseg.cpu().numpy()
        for i in range(3):
            want, wn = oracle.extract_segments(b[0], tuple(pk[0, i]), c, s, fg, ml, cap=8)
            assert nseg[0, i] == wn
            assert [tuple(int(v) for v in segs[0, i, j]) for j in range(min(wn, 8))] == want
    # theta bins outside the table (a sentinel, or peaks of another table
    # size) inside n_peaks: no segments, no out-of-table read
    bad = np.array([[[-1, d, 1], [180, d + 45, 1], [90, d + 45, 1]]], np.int32)
    segs, nseg = ld.extract_segments(cuda(b), cuda(bad), cuda(npk), c, s, 15, 0, 8)
    torch.cuda.synchronize()
    nseg = nseg.cpu().numpy()
    assert nseg[0, 0] == 0 and nseg[0, 1] == 0
    want, wn = oracle.extract_segments(b[0], tuple(bad[0, 2]), c, s, 15, 0, cap=8)
    assert nseg[0, 2] == wn


# ----------------------------------------------------------------------------
# SPEC float64 trig mode (NEXT 4, DESIGN R29) against the oracle, bit-exact
# ----------------------------------------------------------------------------
def _gpu_vote_f64(ld, lists, w, h, c, s):
    b = len(lists)
    stride = ld._round_up(max(max(len(e) for e in lists), 1), 4)
    el = np.zeros((b, stride), np.uint32)
    for i, e in enumerate(lists):
        el[i, :len(e)] = e
    counts = cuda(np.array([len(e) for e in lists], np.int32))
    acc = ld.hough_accumulate_f64(cuda(el.view(np.int32)), counts, stride, w, h, c, s)
    torch.cuda.synchronize()
    return acc.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("n_theta", [1, 2, 3, 180, 181, 720, 1024])
def test_vote_f64_random_lists(ld, oracle, n_theta):
    c, s = synth.f64_table(n_theta)
    rng = np.random.default_rng(500 + n_theta)
    w, h = 301, 203
    lists = []
    for n in (0, 1, 7, 5003):
        xs, ys = rng.integers(0, w, n), rng.integers(0, h, n)
        lists.append(((ys.astype(np.uint32) << 16) | xs.astype(np.uint32)))
    got = _gpu_vote_f64(ld, lists, w, h, c, s)
    for i, e in enumerate(lists):
        assert np.array_equal(got[i], oracle.hough_accumulate_f64(e, w, h, c, s)), (n_theta, i)


def test_vote_f64_frames_and_corners(ld, oracle):
    c, s = synth.f64_table(180)
    img = synth.gen_frame("cfg2", 0)
    _, edges, counts, stride = ld.sobel_binarize(cuda(img[None]), 200, want_binary=False)
    acc = ld.hough_accumulate_f64(edges, counts, stride, 1280, 720, c, s)
    torch.cuda.synchronize()
    e = oracle.compact(oracle.sobel_binarize(img, 200))
    assert np.array_equal(acc.cpu().numpy().view(np.uint32)[0],
                          oracle.hough_accumulate_f64(e, 1280, 720, c, s))
    for w, h in [(1, 1), (16384, 1), (1, 16384), (16384, 16384)]:
        c2, s2 = synth.f64_table(64)
        corners = sorted({(0, 0), (w - 1, 0), (0, h - 1), (w - 1, h - 1)})
        ee = np.array([(y << 16) | x for x, y in corners], np.uint32)
        got = _gpu_vote_f64(ld, [ee], w, h, c2, s2)
        assert np.array_equal(got[0], oracle.hough_accumulate_f64(ee, w, h, c2, s2)), (w, h)


def test_vote_f64_rejects_bad_tables(ld):
    el = torch.zeros((4,), dtype=torch.int32, device="cuda")
    cnt = torch.zeros((1,), dtype=torch.int32, device="cuda")
    acc = torch.zeros((1, 2, 2 * ld.ld_rho_offset(10, 10) + 1), dtype=torch.int32, device="cuda")
    for c, s in [([1.5, 0.0], [0.0, 1.0]), ([float("nan"), 0.0], [0.0, 1.0])]:
        with pytest.raises(ld.LdError) as ei:
            ld.ld_hough_accumulate_f64(el, cnt, 4, 1, 10, 10, 2, c, s, acc)
        assert ei.value.status == ld.LD_ERR_RANGE
    with pytest.raises(ld.LdError):
        ld.ld_hough_accumulate_f64(el, cnt, 4, 1, 10, 10, 1025, [0.0] * 1025, [0.0] * 1025, acc)


def test_hinted_peaks_randomized_stress(ld, oracle):
    # random images x windows (warp, stream, tile and band kernels) x k, the
    # hinted path against the oracle and against the unhinted path
    rng = np.random.default_rng(777)
    for trial in range(10):
        b = int(rng.integers(1, 5))
        w, h = int(rng.integers(40, 300)), int(rng.integers(20, 200))
        frames = np.zeros((b, h, w), np.uint8)
        for f in range(b):
            frames[f] = (rng.random((h, w)) < rng.uniform(0.02, 0.3)) * 255
            for _ in range(int(rng.integers(0, 4))):
                y = int(rng.integers(0, h))
                frames[f, y, :] = 255
        n_theta = int(rng.choice([90, 180, 181]))
        ht = int(rng.choice([0, 1, 2, 3, 5, 8, 13]))
        hr = int(rng.choice([4, 9, 29, 64, 70]))
        k = int(rng.choice([1, 3, 4, 16, 64, 100]))
        cfg = synth.Config("t", w, h, b, 200, n_theta, k, ht, hr)
        _hint_case(ld, oracle, frames, cfg)


def test_detect_randomized_soak(ld, oracle):
    # end to end through ld_detect_batch (paired voting + peak hint inside)
    # on random images, thresholds, theta counts, windows and k
    rng = np.random.default_rng(4242)
    for trial in range(12):
        b = int(rng.integers(1, 4))
        w, h = int(rng.integers(3, 400)), int(rng.integers(3, 300))
        frames = rng.integers(0, 256, size=(b, h, w)).astype(np.uint8)
        if trial % 3 == 0:
            frames = (frames > 200).astype(np.uint8) * 255
        thr = int(rng.choice([1, 100, 200, 700, 1531]))
        n_theta = int(rng.choice([1, 2, 7, 90, 180, 181, 360]))
        c, s = synth.q15_table(n_theta)
        ht, hr = int(rng.integers(0, 8)), int(rng.integers(0, 70))
        mv, k = int(rng.integers(0, 6)), int(rng.choice([1, 2, 4, 16, 64]))
        peaks, npk, counts, acc = ld.detect_batch(cuda(frames), thr, c, s, ht, hr, mv, k)
        torch.cuda.synchronize()
        P, N, C, A = (peaks.cpu().numpy(), npk.cpu().numpy(), counts.cpu().numpy(),
                      acc.cpu().numpy().view(np.uint32))
        for f in range(b):
            r = oracle.detect(frames[f], thr, c, s, ht, hr, mv, k)
            assert int(C[f]) == r["n_edges"], (trial, f)
            assert np.array_equal(A[f], r["acc"]), (trial, f)
            assert int(N[f]) == r["n_peaks"], (trial, f)
            assert peak_tuples(P[f]) == oracle_peak_tuples(r["peaks"]), (trial, f)


def test_pipelined_detector_matches_single_stream(ld, oracle):
    cfg = synth.CONFIGS["cfg3"]
    c, s = synth.q15_table(cfg.n_theta)
    frames = [synth.gen_batch("cfg3", 8 * i, 8) for i in range(5)]
    pd = ld.PipelinedDetector(1280, 720, 8, cfg.n_theta, c, s, cfg.threshold, cfg.k,
                              cfg.half_theta, cfg.half_rho, cfg.min_votes, streams=3)
    # more batches than slots in flight, no host synchronisation in between:
    # each input is a fresh tensor dropped right after submit (the caching
    # allocator may hand its block to the next allocation -- submit() must
    # have recorded the slot's stream on it), and the outputs are copied on
    # the current stream after the slot's event (a slot is reused 3 submits
    # later, after this stream's copies: submit() orders it after them)
    outs = []
    for f in frames:
        g = cuda(f)  # 1280 is a multiple of 16: pitch == width
        pk, npk, cnt, ev = pd.submit(g)
        del g
        junk = torch.full((8, 720, 1280), 255, dtype=torch.uint8, device="cuda")
        del junk
        torch.cuda.current_stream().wait_event(ev)
        outs.append((pk.clone(), npk.clone(), cnt.clone()))
    torch.cuda.synchronize()
    for i, f in enumerate(frames):
        ref = ld.detect_batch(cuda(f), cfg.threshold, c, s, cfg.half_theta, cfg.half_rho,
                              cfg.min_votes, cfg.k, export_acc=False)
        torch.cuda.synchronize()
        assert torch.equal(outs[i][0], ref[0]) and torch.equal(outs[i][1], ref[1])
        assert torch.equal(outs[i][2], ref[2])
    r = oracle.detect(frames[2][3], cfg.threshold, c, s, cfg.half_theta, cfg.half_rho,
                      cfg.min_votes, cfg.k, want_binary=False, want_acc=False)
    assert peak_tuples(outs[2][0][3].cpu()) == oracle_peak_tuples(r["peaks"])


def test_detect_is_cuda_graph_capturable(ld):
    # the C ABI enqueues without host synchronisation: a whole detect step
    # captures into a CUDA graph and replays to the same result
    cfg = synth.CONFIGS["cfg3"]
    c, s = synth.q15_table(cfg.n_theta)
    g = cuda(synth.gen_batch("cfg3", 0, 4))
    det = ld.Detector(1280, 720, 4, cfg.n_theta, c, s, cfg.threshold, cfg.k, cfg.half_theta,
                      cfg.half_rho, cfg.min_votes)
    ref = [t.clone() for t in det(g)[:3]]
    torch.cuda.synchronize()
    for t in (det.peaks, det.n_peaks, det.counts):
        t.fill_(-7)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        det(g, torch.cuda.current_stream())
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(det.peaks, ref[0]) and torch.equal(det.n_peaks, ref[1])
    assert torch.equal(det.counts, ref[2])


@pytest.mark.parametrize("name,n_theta", [("cfg1", 16), ("cfg2", 32), ("cfg2", 48), ("cfg1", 180)])
def test_vote_cluster_split_equals_single_cta(ld, oracle, name, n_theta):
    """Launches whose one-pair bands still leave most SMs idle (single frames
    with few theta bins) vote through thread-block clusters (a band's edges
    split over the cluster's CTAs, copies summed over distributed shared
    memory): the accumulator, the chunk maxima and the hinted peaks equal the
    one-CTA-per-band path and the oracle.  (A full 180-bin table on a single
    frame fills the GPU with one-pair bands: no cluster.)"""
    cfg = synth.CONFIGS[name]
    cfg = synth.Config(cfg.name, cfg.width, cfg.height, 1, cfg.threshold, n_theta, cfg.k,
                       cfg.half_theta, cfg.half_rho)
    c, s = synth.q15_table(cfg.n_theta)
    img = synth.gen_frame(name, 0)
    _, edges, counts, stride = ld.sobel_binarize(cuda(img[None]), cfg.threshold,
                                                 want_binary=False)
    h, w = img.shape
    a_cl, h_cl = ld.hough_accumulate(edges, counts, stride, w, h, c, s, want_hint=True)
    a_1, h_1 = ld.hough_accumulate(edges, counts, stride, w, h, c, s, want_hint=True,
                                   flags=ld.LD_VOTE_NO_CLUSTER)
    torch.cuda.synchronize()
    assert torch.equal(a_cl, a_1)
    # hint header word 5 = keys per band: one per CTA of a cluster (G = 8
    # here), one per warp (16) without
    kpb = int(h_cl[:64].view(torch.int32)[5].item()), int(h_1[:64].view(torch.int32)[5].item())
    assert kpb == ((16, 16) if n_theta == 180 else (8, 16)), kpb
    want = oracle.hough_accumulate(oracle.compact(oracle.sobel_binarize(img, cfg.threshold)),
                                   w, h, c, s)
    assert np.array_equal(a_cl.cpu().numpy().view(np.uint32)[0], want)
    check_chunk_maxima(a_cl, h_cl)
    p0, n0 = ld.hough_peaks(a_cl, cfg.half_theta, cfg.half_rho, 1, cfg.k)
    p1, n1 = ld.hough_peaks(a_cl, cfg.half_theta, cfg.half_rho, 1, cfg.k, hint=h_cl)
    assert torch.equal(p0, p1) and torch.equal(n0, n1)
