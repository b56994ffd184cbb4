"""Multi-GPU host logic on CPU: partitions, and the
row-band exchange step through a real world-size-2 gloo process group.

The banded path's arithmetic is libld.so's (GPU, covered by
test_gpu_parity.py::test_banded_*); here each rank computes its band with the
ORACLE on the band's own rows (1-row halo, exactly what ld_image.row_begin /
row_end hand to the kernel), so these tests check the partition, the halo
convention, global coordinates and the exact int32 SUM of uint32 accumulators
against the whole-image oracle.
"""
import os
import socket

import numpy as np
import pytest

from paper_2212_09460_b200 import dist as pdist
from paper_2212_09460_b200 import synth


@pytest.mark.parametrize("world", [1, 2, 3, 4, 5, 8])
def test_frame_shards_cover_exactly(world):
    for n in (0, 1, 7, 64, 256, 257):
        seen = []
        for r in range(world):
            first, cnt = pdist.frame_shard(n, r, world)
            seen.extend(range(first, first + cnt))
            assert cnt in (n // world, n // world + 1)
        assert seen == list(range(n))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_row_bands_and_halo(world):
    for h in (1, 2, 3, 5, 240, 4096):
        rows = []
        for r in range(world):
            p = pdist.BandPlan.make(100, h, r, world)
            rows.extend(range(p.row_begin, p.row_end))
            if p.rows:
                assert p.read_begin == max(p.row_begin - 1, 0)
                assert p.read_end == min(p.row_end + 1, h)
                assert p.max_edges == p.rows * 98
        assert rows == list(range(h))


def band_accumulator(oracle, img, plan, c, s):
    """Oracle on the band's rows only (what the kernel sees), edges in global y."""
    if plan.rows == 0:
        return np.zeros((len(c), 2 * oracle.rho_offset(plan.width, plan.height) + 1), np.uint32)
    sub = img[plan.read_begin:plan.read_end]
    b = oracle.sobel_binarize(sub, 200)
    off = plan.row_begin - plan.read_begin
    own = np.zeros_like(b)
    own[off:off + plan.rows] = b[off:off + plan.rows]
    # rows that are global borders are 0 in the sub-image too (they are its
    # first/last row); interior band rows are interior rows of the sub-image
    e = oracle.compact(own).astype(np.int64)
    y = (e >> 16) + plan.read_begin
    x = e & 0xFFFF
    eg = ((y << 16) | x).astype(np.uint32)
    return oracle.hough_accumulate(eg, plan.width, plan.height, c, s)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img = synth.random_image(5, 96, 67, "uniform")
        c, s = synth.q15_table(90)
        plan = pdist.BandPlan.make(96, 67, rank, world)
        acc = band_accumulator(oracle, img, plan, c, s)
        t = torch.from_numpy(acc.view(np.int32).copy())
        pdist.allreduce_accumulator(t)
        summed = t.numpy().view(np.uint32)
        pk, npk = oracle.hough_peaks(summed, 2, 6, 1, 8)
        np.save(os.path.join(outdir, "acc%d.npy" % rank), summed)
        np.save(os.path.join(outdir, "pk%d.npy" % rank),
                np.array([(p["theta_bin"], p["rho_bin"], p["votes"]) for p in pk], np.int64))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_banded_allreduce_gloo_equals_whole_oracle(oracle, tmp_path, world):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    img = synth.random_image(5, 96, 67, "uniform")
    c, s = synth.q15_table(90)
    want = oracle.hough_accumulate(oracle.compact(oracle.sobel_binarize(img, 200)), 96, 67, c, s)
    wpk, _ = oracle.hough_peaks(want, 2, 6, 1, 8)
    wpk = np.array([(p["theta_bin"], p["rho_bin"], p["votes"]) for p in wpk], np.int64)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / ("acc%d.npy" % r)), want), r
        assert np.array_equal(np.load(tmp_path / ("pk%d.npy" % r)), wpk), r


def test_band_accumulators_sum_to_whole_without_collective(oracle):
    # the same additivity, all bands in one process, for several world sizes
    # including more ranks than rows
    img = synth.random_image(9, 40, 6, "uniform")
    c, s = synth.q15_table(32)
    want = oracle.hough_accumulate(oracle.compact(oracle.sobel_binarize(img, 200)), 40, 6, c, s)
    for world in (1, 2, 4, 8):
        tot = sum(band_accumulator(oracle, img, pdist.BandPlan.make(40, 6, r, world), c, s)
                  .astype(np.int64) for r in range(world))
        assert np.array_equal(tot, want.astype(np.int64)), world


# ----------------------------------------------------------------------------
# theta-sharded detection (NEXT 1): partition, halo slices and the exchange of
# per-shard top-k lists through a real gloo process group
# ----------------------------------------------------------------------------
def test_theta_slices_cover_with_halo():
    for nt, ht in [(180, 2), (1024, 10), (7, 3), (3, 0)]:
        for world in (1, 2, 3, 8):
            owned = []
            for r in range(world):
                t0, t1 = pdist.theta_shard(nt, r, world)
                g0, g1 = pdist.theta_slice(nt, ht, t0, t1)
                owned.extend(range(t0, t1))
                assert g0 == max(t0 - ht, 0) and g1 == min(t1 + ht, nt)
            assert owned == list(range(nt))


def _shard_peaks(oracle, big, t0, t1, ht, hr, k):
    g0, g1 = pdist.theta_slice(big.shape[0], ht, t0, t1)
    sl = np.ascontiguousarray(big[g0:g1])
    pk, _ = oracle.hough_peaks(sl, ht, hr, 1, sl.size)  # every candidate of the slice
    own = [(int(p["theta_bin"]) + g0, int(p["rho_bin"]), int(p["votes"])) for p in pk
           if t0 - g0 <= int(p["theta_bin"]) < t1 - g0][:k]
    out = np.full((k, 3), -1, np.int32)
    out[:, 2] = 0
    for i, t in enumerate(own):
        out[i] = t
    return out, len(own)


def _merge_by_key(peaks, n_peaks, n_rho, k):
    """Top k of the per-shard lists by (votes, -theta, -rho) (DESIGN R14)."""
    keys = [(int(v), -(int(t) * n_rho + int(r)), int(t), int(r))
            for lst, n in zip(peaks, n_peaks) for (t, r, v) in lst[:int(n)]]
    keys.sort(reverse=True)
    out = np.full((k, 3), -1, np.int32)
    out[:, 2] = 0
    for i, (v, _, t, r) in enumerate(keys[:k]):
        out[i] = (t, r, v)
    return out, min(k, len(keys))


def _theta_worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img = synth.random_image(17, 90, 70, "uniform")
        c, s = synth.q15_table(60)
        e = oracle.compact(oracle.sobel_binarize(img, 300))
        big = oracle.hough_accumulate(e, 90, 70, c, s)
        t0, t1 = pdist.theta_shard(60, rank, world)
        p, n = _shard_peaks(oracle, big, t0, t1, 2, 5, 6)
        allp = [torch.zeros((6, 3), dtype=torch.int32) for _ in range(world)]
        alln = [torch.zeros((1,), dtype=torch.int32) for _ in range(world)]
        dist.all_gather(allp, torch.from_numpy(p))
        dist.all_gather(alln, torch.tensor([n], dtype=torch.int32))
        # the merge itself is libld's ld_merge_peak_lists (GPU, test_gpu_parity);
        # here the gathered lists merge by the same key in plain Python
        mp, mn = _merge_by_key(torch.stack(allp).numpy(), torch.cat(alln).numpy(),
                               big.shape[1], 6)
        np.save(os.path.join(outdir, "tp%d.npy" % rank), mp)
        np.save(os.path.join(outdir, "tn%d.npy" % rank), np.array([mn], np.int32))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_theta_sharded_merge_gloo_equals_whole_oracle(oracle, tmp_path, world):
    import torch.multiprocessing as mp
    mp.spawn(_theta_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    img = synth.random_image(17, 90, 70, "uniform")
    c, s = synth.q15_table(60)
    big = oracle.hough_accumulate(oracle.compact(oracle.sobel_binarize(img, 300)), 90, 70, c, s)
    want, wn = oracle.hough_peaks(big, 2, 5, 1, 6)
    want = np.array([(p["theta_bin"], p["rho_bin"], p["votes"]) for p in want], np.int64)
    for r in range(world):
        got = np.load(tmp_path / ("tp%d.npy" % r)).astype(np.int64)
        assert int(np.load(tmp_path / ("tn%d.npy" % r))[0]) == wn
        assert np.array_equal(got[:wn], want[:wn]) and (got[wn:, 0] == -1).all(), r
