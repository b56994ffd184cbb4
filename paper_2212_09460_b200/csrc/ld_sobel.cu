// ld_sobel.cu -- B1: fused Sobel |Gx|+|Gy| + binarize + edge compaction, sm_100a.
//
// Paper: Eq. 1 with the Fig. 2 kernels, binarization to
// {0,255}, per-pixel GPU mapping, and the edge
// coordinate list read by the voting blocks.  DESIGN.md section 6.1.
//
// Design (B200-first, not the paper's K80 design):
//  * Persistent CTAs (3 per SM) walk a frame-major list of 64 x 224 output
//    tiles.  Each tile's input (66 x 256 bytes: 1-row halo above/below, 16
//    columns left, 16 right) is staged by a TMA 3-D box load into a 4-deep
//    shared-memory ring completed on mbarriers, so HBM reads of later tiles
//    overlap the arithmetic of the current one.  Out-of-image halo bytes are
//    zero-filled by TMA and only ever feed border pixels, which are forced to 0.
//  * Arithmetic: |Gx|+|Gy| = 2 max(|A|, |B|) with
//      A = (p01+p02+p12) - (p10+p20+p21),  B = (p12+p21+p22) - (p00+p01+p10)
//    (pRC = row R of y-1..y+1, column C of x-1..x+1), an exact identity
//    (|a|+|b| = max(|a+b|, |a-b|), Gx+Gy = 2A, Gx-Gy = 2B).  The test
//    |Gx|+|Gy| >= T becomes max(|A|,|B|) >= T2 = ceil(T/2).  Two pixels are
//    processed per 32-bit register as 16-bit lanes (SWAR): each lane of
//    A + 2048 - T2 lies in [517, 2813], so bit 11 of each half is the
//    comparison result and no carry ever crosses a half.
//  * Compaction: per-thread popcount, a CTA scan in 16x16-cell order, one
//    counter reservation (atomicAdd on the frame's edge counter) per tile,
//    whose round trip is hidden by writing each tile's edges one iteration
//    late.  The cell order makes every 32 consecutive list entries spatially
//    compact: the voting kernel's warps then hit few, consecutive rho bins
//    (distinct shared-memory banks; same-bin lanes merge in ATOMS.POPC.INC).
#include "ld_internal.cuh"

namespace ld {

struct RowV {
  uint32_t E[4];   // halves: pixels (4k, 4k+2)
  uint32_t O[4];   // halves: pixels (4k+1, 4k+3)
  uint32_t OL[4];  // halves: pixels (4k-1, 4k+1)
  uint32_t ER[4];  // halves: pixels (4k+2, 4k+4)
};

// p points at the chunk's first byte in a staged shared-memory row.
__device__ __forceinline__ void load_row(const uint8_t *p, RowV &r) {
  const uint4 w = *reinterpret_cast<const uint4 *>(p);
  const uint32_t wl = *reinterpret_cast<const uint32_t *>(p - 4);
  const uint32_t wr = *reinterpret_cast<const uint32_t *>(p + 16);
  const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
  uint32_t om1 = prmt(wl, 0u, 0x4341u);
  uint32_t e4 = prmt(wr, 0u, 0x4240u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    r.E[k] = prmt(ww[k], 0u, 0x4240u);
    r.O[k] = prmt(ww[k], 0u, 0x4341u);
  }
  r.OL[0] = prmt(om1, r.O[0], 0x5432u);
#pragma unroll
  for (int k = 1; k < 4; ++k) r.OL[k] = prmt(r.O[k - 1], r.O[k], 0x5432u);
#pragma unroll
  for (int k = 0; k < 3; ++k) r.ER[k] = prmt(r.E[k], r.E[k + 1], 0x5432u);
  r.ER[3] = prmt(r.E[3], e4, 0x5432u);
}

__device__ __forceinline__ uint32_t flag2(uint32_t pa, uint32_t na, uint32_t pb, uint32_t nb,
                                          uint32_t k0) {
  const uint32_t x1 = pa - na + k0, x2 = na - pa + k0;
  const uint32_t y1 = pb - nb + k0, y2 = nb - pb + k0;
  return (x1 | x2 | y1 | y2) & 0x08000800u;
}

// One output row of 16 pixels.  Returns the edge mask with bit (8j + k) set for
// pixel 4k + j; outw[k] receives the binary bytes of pixels 4k..4k+3.
__device__ __forceinline__ uint32_t sobel_row(const RowV &u, const RowV &m, const RowV &d,
                                              uint32_t k0, const uint32_t colb[4],
                                              uint32_t outw[4]) {
  uint32_t all = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    // even pixels 4k, 4k+2: L = OL, C = E, R = O
    const uint32_t fe = flag2(u.E[k] + u.O[k] + m.O[k], d.OL[k] + d.E[k] + m.OL[k],
                              d.E[k] + d.O[k] + m.O[k], u.OL[k] + u.E[k] + m.OL[k], k0);
    // odd pixels 4k+1, 4k+3: L = E, C = O, R = ER
    const uint32_t fo = flag2(u.O[k] + u.ER[k] + m.ER[k], d.E[k] + d.O[k] + m.E[k],
                              d.O[k] + d.ER[k] + m.ER[k], u.E[k] + u.O[k] + m.E[k], k0);
    const uint32_t bits = ((fe >> 11) | (fo >> 3)) & colb[k];  // 0/1 per byte
    outw[k] = bits * 255u;
    all |= bits << k;
  }
  return all;
}

__device__ __forceinline__ void write_edges(const SobelParams &p, const uint32_t masks[SB_SR],
                                            int f, int ybase, int xs, uint32_t off) {
  uint32_t *dst = p.edges + static_cast<int64_t>(f) * p.edge_stride + off;
#pragma unroll
  for (int i = 0; i < SB_SR; ++i) {
    uint32_t m = masks[i];
    const uint32_t yy = static_cast<uint32_t>(ybase + i) << 16;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      *dst++ = yy | static_cast<uint32_t>(xs + 4 * (b & 7) + (b >> 3));
    }
  }
}

__global__ void __launch_bounds__(SB_THREADS, SB_CTAS_PER_SM)
    sobel_binarize_compact_kernel(const __grid_constant__ CUtensorMap tmap,
                                  const SobelParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~static_cast<uintptr_t>(127));
  constexpr int NW = SB_THREADS / 32;
  __shared__ __align__(8) uint64_t full_bar[SB_STAGES];
  __shared__ uint32_t s_cnt[SB_THREADS];        // per-thread counts, in cell order
  __shared__ uint32_t s_excl[2][SB_THREADS];    // exclusive scan inside each warp
  __shared__ uint32_t s_wt[NW];                 // warp totals
  __shared__ uint32_t s_wbase[2][NW];           // exclusive scan of warp totals
  __shared__ uint32_t s_base[2];                // frame-list base of the tile

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int chunk = tid % SB_CHUNKS;
  const int strip = tid / SB_CHUNKS;
  // List order inside a tile: 16x16-pixel cells (4 strips of one chunk), cells
  // row-major.  32 consecutive list entries then span a compact region, so a
  // warp of the voting kernel hits <= ~32 consecutive rho bins per theta.
  const int ord = ((strip >> 2) * SB_CHUNKS + chunk) * 4 + (strip & 3);
  const uint32_t k0 = static_cast<uint32_t>(2048 - p.t2) * 0x00010001u;

  auto issue = [&](int tile, int stage) {
    const int f = tile / p.tiles_per_frame;
    const int rem = tile - f * p.tiles_per_frame;
    const int ty = rem / p.tiles_x;
    const int tx = rem - ty * p.tiles_x;
    const int y = p.row_begin + ty * SB_TILE_H - 1 - p.ry0;  // tensor row of smem row 0
    const int x = tx * SB_TILE_W - SB_HALO_L;
    mbar_arrive_expect_tx(&full_bar[stage], SB_STAGE_BYTES);
    tma_load_3d(smem + stage * SB_STAGE_BYTES, &tmap, &full_bar[stage], x, y, f);
  };

  if (tid == 0) {
    for (int s = 0; s < SB_STAGES; ++s) mbar_init(&full_bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < SB_STAGES; ++s) {
      const int tile = blockIdx.x + s * gridDim.x;
      if (tile < p.n_tiles) issue(tile, s);
    }
  }

  // previous tile, written one iteration late so that the counter
  // reservation (a global atomic round trip) overlaps the next tile's work
  uint32_t pmask[SB_SR] = {0u, 0u, 0u, 0u};
  int pf = 0, pybase = 0, pxs = 0;
  uint32_t base_reg = 0;  // thread 0: reservation result of the previous tile

  int it = 0;
  for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++it) {
    const int stage = it % SB_STAGES;
    const uint32_t parity = (it / SB_STAGES) & 1;
    const int cb = it & 1, pb = cb ^ 1;
    const int f = tile / p.tiles_per_frame;
    const int rem = tile - f * p.tiles_per_frame;
    const int ty = rem / p.tiles_x;
    const int tx = rem - ty * p.tiles_x;
    const int y0 = p.row_begin + ty * SB_TILE_H;  // first output row of the tile
    const int xs = tx * SB_TILE_W + chunk * 16;   // first column of this thread's chunk

    // interior-column bytes (0x01 per pixel with 1 <= x <= W-2)
    uint32_t colb[4];
    {
      const int lo = 1 - xs, hi = p.width - 2 - xs;  // valid j in [lo, hi]
      if (lo <= 0 && hi >= 15) {
#pragma unroll
        for (int k = 0; k < 4; ++k) colb[k] = 0x01010101u;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t b = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int jj = 4 * k + j;
            if (jj >= lo && jj <= hi) b |= 1u << (8 * j);
          }
          colb[k] = b;
        }
      }
    }

    mbar_wait(&full_bar[stage], parity);
    const uint8_t *buf = smem + stage * SB_STAGE_BYTES + SB_HALO_L + chunk * 16;

    uint32_t masks[SB_SR];
    const int ybase = y0 + strip * SB_SR;  // output row of masks[0]
    {
      RowV r0, r1, r2;
      load_row(buf + (strip * SB_SR + 0) * SB_BOX_W, r0);
      load_row(buf + (strip * SB_SR + 1) * SB_BOX_W, r1);
#pragma unroll
      for (int i = 0; i < SB_SR; ++i) {
        load_row(buf + (strip * SB_SR + i + 2) * SB_BOX_W, r2);
        const int y = ybase + i;
        const bool owned = y < p.row_end;
        const bool interior = y >= 1 && y <= p.height - 2 && owned;
        uint32_t outw[4] = {0u, 0u, 0u, 0u};
        uint32_t all = 0;
        if (interior) all = sobel_row(r0, r1, r2, k0, colb, outw);
        masks[i] = all;
        if (p.binary != nullptr && owned && xs < p.width) {
          uint8_t *dst = p.binary + static_cast<int64_t>(f) * p.bin_frame_stride +
                         static_cast<int64_t>(y - p.row_begin) * p.bin_pitch + xs;
          *reinterpret_cast<uint4 *>(dst) = make_uint4(outw[0], outw[1], outw[2], outw[3]);
        }
        r0 = r1;
        r1 = r2;
      }
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < SB_SR; ++i) cnt += __popc(masks[i]);
    s_cnt[ord] = cnt;
    if (tid == 0 && it > 0) s_base[pb] = base_reg;
    __syncthreads();  // (A): stage consumed, counts and previous base visible
    if (tid == 0) {
      const int next = tile + SB_STAGES * gridDim.x;
      if (next < p.n_tiles) issue(next, stage);
    }
    if (it > 0 && p.edges != nullptr) {
      const uint32_t off = s_base[pb] + s_wbase[pb][ord >> 5] + s_excl[pb][ord];
      write_edges(p, pmask, pf, pybase, pxs, off);
    }
    {  // scan of this tile's counts in cell order
      const uint32_t x = s_cnt[tid];
      uint32_t incl = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      s_excl[cb][tid] = incl - x;
      if (lane == 31) s_wt[warp] = incl;
    }
    __syncthreads();  // (B)
    if (tid == 0) {
      uint32_t acc = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        s_wbase[cb][w] = acc;
        acc += s_wt[w];
      }
      base_reg = acc ? atomicAdd(&p.counts[f], acc) : 0u;  // consumed next iteration
    }
#pragma unroll
    for (int i = 0; i < SB_SR; ++i) pmask[i] = masks[i];
    pf = f;
    pybase = ybase;
    pxs = xs;
  }
  if (it > 0) {
    const int pb = (it - 1) & 1;
    if (tid == 0) s_base[pb] = base_reg;
    __syncthreads();
    if (p.edges != nullptr) {
      const uint32_t off = s_base[pb] + s_wbase[pb][ord >> 5] + s_excl[pb][ord];
      write_edges(p, pmask, pf, pybase, pxs, off);
    }
  }
}

cudaError_t launch_sobel(const CUtensorMap &tmap, const SobelParams &p, int n_ctas,
                         cudaStream_t stream) {
  const size_t smem = static_cast<size_t>(SB_STAGES) * SB_STAGE_BYTES + 128;
  static bool attr_done[64];  // idempotent per-device attribute; benign race
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_done[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(sobel_binarize_compact_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr_done[dev & 63] = true;
  }
  sobel_binarize_compact_kernel<<<n_ctas, SB_THREADS, smem, stream>>>(tmap, p);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ld
