"""Full-batch parity at BASELINE.json's own sizes and launch configurations.

Every frame of cfg3 (256 x 1280x720) and cfg4 (64 x 1920x1080) goes through
the GPU in ONE launch sequence -- both ld_detect_batch (the fused entry
point) and the benchmark's step (ld_sobel_binarize -> ld_hough_accumulate_hint
-> ld_hough_peaks_hinted on their own buffers) -- and every frame's edge
count, edge set, accumulator and peaks are compared with the CPU oracle,
frame-parallel over the host cores (oracle.parity).  cfg5 is compared whole
for the row-band (N = 2/4/8) and theta-shard (N = 2/4/8) decompositions,
every rank emulated in one process.  Expected values come only from oracle/.
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


def _upload(ld, frames):
    b, h, w = frames.shape
    pitch = ld._round_up(w, 16)
    g = torch.zeros((b, h, pitch), dtype=torch.uint8, device="cuda")
    g[:, :, :w] = torch.from_numpy(frames).cuda()
    return g, pitch


def _bench_step(ld, name, frames):
    """The benchmark's step (bench.py run_ours) on the whole batch."""
    cfg = synth.CONFIGS[name]
    c, s = synth.q15_table(cfg.n_theta)
    b, h, w = frames.shape
    g, pitch = _upload(ld, frames)
    img = ld.make_image(w, h, pitch, h * pitch, b)
    stride = ld._round_up(h * max(w - 2, 0), 4)
    n_rho = 2 * ld.ld_rho_offset(w, h) + 1
    edges = torch.full((b, stride), -1, dtype=torch.int32, device="cuda")
    counts = torch.full((b,), -1, dtype=torch.int32, device="cuda")
    acc = torch.full((b, cfg.n_theta, n_rho), -1, dtype=torch.int32, device="cuda")
    hb = ld.ld_hough_hint_bytes(b, w, h, cfg.n_theta)
    hint = torch.empty((hb,), dtype=torch.uint8, device="cuda")
    wb = ld.ld_hough_peaks_workspace_bytes(b, cfg.n_theta, n_rho, cfg.k)
    ws = torch.empty((wb,), dtype=torch.uint8, device="cuda")
    peaks = torch.full((b, cfg.k, 3), 7, dtype=torch.int32, device="cuda")
    npk = torch.full((b,), -7, dtype=torch.int32, device="cuda")
    ld.ld_sobel_binarize(g, img, cfg.threshold, None, edges, stride, counts)
    ld.ld_hough_accumulate_hint(edges, counts, stride, b, w, h, cfg.n_theta, c, s, acc, hint, hb)
    ld.ld_hough_peaks_hinted(acc, b, cfg.n_theta, n_rho, cfg.half_theta, cfg.half_rho,
                             cfg.min_votes, cfg.k, hint, hb, peaks, npk, ws, wb)
    torch.cuda.synchronize()
    return edges, counts, acc, peaks, npk


def _check_all(oracle, name, frames, counts, acc, peaks, npk, edges=None):
    from oracle import parity
    cfg = synth.CONFIGS[name]
    c, s = synth.q15_table(cfg.n_theta)
    cnt = counts.cpu().numpy()
    pk = peaks.cpu().numpy()
    npk_h = npk.cpu().numpy()

    def get(f):
        a = acc[f].cpu().numpy()
        e = None if edges is None else edges[f, : int(cnt[f])].cpu().numpy().view(np.uint32)
        return cnt[f], pk[f], npk_h[f], a, e

    r = parity.check_batch(frames, cfg.threshold, c, s, cfg.half_theta, cfg.half_rho,
                           cfg.min_votes, cfg.k, get)
    assert r["ok"], "%d/%d frames differ; first: %s" % (r["mismatches"], r["frames"],
                                                        r["first_mismatch"])
    return r


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_bench_step_every_frame(ld, oracle, name):
    frames = synth.gen_batch(name)
    assert frames.shape[0] == synth.CONFIGS[name].batch
    edges, counts, acc, peaks, npk = _bench_step(ld, name, frames)
    _check_all(oracle, name, frames, counts, acc, peaks, npk, edges)


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_detect_batch_every_frame(ld, oracle, name):
    cfg = synth.CONFIGS[name]
    c, s = synth.q15_table(cfg.n_theta)
    frames = synth.gen_batch(name)
    b, h, w = frames.shape
    det = ld.Detector(w, h, b, cfg.n_theta, c, s, cfg.threshold, cfg.k, cfg.half_theta,
                      cfg.half_rho, cfg.min_votes, export_acc=True)
    g, _ = _upload(ld, frames)
    peaks, npk, counts, acc = det(g)
    torch.cuda.synchronize()
    _check_all(oracle, name, frames, counts, acc, peaks, npk)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("shard", ["band", "theta"])
def test_cfg5_decompositions_whole_image(ld, oracle, world, shard):
    """cfg5 at N = 2/4/8, every rank emulated in this process (no process
    group): the row-band partial accumulators summed (what the NCCL all_reduce
    computes) and the theta-shard top-k merge, against the whole-image oracle
    (edge count, accumulator, peaks)."""
    from paper_2212_09460_b200 import dist as pdist
    cfg = synth.CONFIGS["cfg5"]
    c, s = synth.q15_table(cfg.n_theta)
    img = synth.gen_frame("cfg5", 0)
    W, H = cfg.width, cfg.height
    want = oracle.detect(img, cfg.threshold, c, s, cfg.half_theta, cfg.half_rho,
                         cfg.min_votes, cfg.k, want_binary=False)
    wp = [(int(p["theta_bin"]), int(p["rho_bin"]), int(p["votes"]))
          for p in want["peaks"][: want["n_peaks"]]]
    bands = []
    for rank in range(world):
        det = pdist.BandedDetector(W, H, cfg.n_theta, c, s, cfg.threshold, cfg.k,
                                   cfg.half_theta, cfg.half_rho, cfg.min_votes, rank, world)
        det.load(img)
        bands.append(det)
    if shard == "band":
        total = None
        for det in bands:
            det()  # no process group: the all_reduce is the identity
            part = det.acc.clone()
            total = part if total is None else total + part
        torch.cuda.synchronize()
        assert sum(int(d.count.item()) for d in bands) == want["n_edges"]
        assert np.array_equal(total.cpu().numpy().view(np.uint32)[0], want["acc"])
        pk, n = ld.hough_peaks(total, cfg.half_theta, cfg.half_rho, cfg.min_votes, cfg.k)
        got = [tuple(int(v) for v in p) for p in pk[0].cpu().numpy()[: int(n[0])]]
        got = [(a, b, int(np.uint32(np.int32(v)))) for a, b, v in got]
    else:
        # the band edge lists, concatenated: what the all_gather delivers
        for det in bands:
            ld.ld_sobel_binarize(det.gray, det.img, cfg.threshold, None, det.edges,
                                 det.edge_stride, det.count)
        torch.cuda.synchronize()
        cl = [int(d.count.item()) for d in bands]
        assert sum(cl) == want["n_edges"]
        edges = torch.cat([d.edges[:n] for d, n in zip(bands, cl)])
        stride = ld._round_up(max(edges.numel(), 1), 4)
        el = torch.zeros((stride,), dtype=torch.int32, device="cuda")
        el[: edges.numel()] = edges
        cnt = torch.tensor([edges.numel()], dtype=torch.int32, device="cuda")
        allp, alln = [], []
        for rank in range(world):
            det = pdist.ThetaShardedDetector(W, H, cfg.n_theta, c, s, cfg.threshold, cfg.k,
                                             cfg.half_theta, cfg.half_rho, cfg.min_votes,
                                             rank, world)
            det.vote_and_peaks(el, cnt, stride)
            allp.append(det.peaks[0].clone())
            alln.append(det.n_peaks.clone())
        p, n = pdist.merge_peak_lists(torch.stack(allp), torch.cat(alln), det.n_rho, cfg.k)
        torch.cuda.synchronize()
        got = [(int(a), int(b), int(np.uint32(np.int32(v))))
               for a, b, v in p.cpu().numpy().reshape(-1, 3)[: int(n.reshape(-1)[0])]]
    assert got == wp
