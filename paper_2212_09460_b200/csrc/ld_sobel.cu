// ld_sobel.cu -- B1: fused Sobel |Gx|+|Gy| + binarize + edge compaction, sm_100a.
//
// Paper: Eq. 1 with the Fig. 2 kernels, binarization to
// {0,255}, per-pixel GPU mapping, and the edge
// coordinate list read by the voting blocks.  DESIGN.md section 6.1.
//
// Design (B200-first, not the paper's K80 design):
//  * Persistent CTAs (3 per SM) walk a frame-major list of 128 x 224 output
//    tiles.  Each tile's input (130 x 256 bytes: 1-row halo above/below, 16
//    columns left, 16 right) is staged by a TMA 3-D box load into a 2-deep
//    shared-memory ring completed on mbarriers, so HBM reads of later tiles
//    overlap the arithmetic of the current one.  Out-of-image halo bytes are
//    zero-filled by TMA and only ever feed border pixels, which are forced to 0.
//  * Arithmetic: |Gx|+|Gy| = 2 max(|A|, |B|) with
//      A = (p01+p02+p12) - (p10+p20+p21),  B = (p12+p21+p22) - (p00+p01+p10)
//    (pRC = row R of y-1..y+1, column C of x-1..x+1), an exact identity
//    (|a|+|b| = max(|a+b|, |a-b|), Gx+Gy = 2A, Gx-Gy = 2B).  The test
//    |Gx|+|Gy| >= T becomes max(|A|,|B|) >= T2 = ceil(T/2).  Two pixels are
//    processed per 32-bit register as 16-bit lanes (SWAR): each lane of
//    A + 2^15 - T2 lies in [2^15 - 1531, 2^15 + 765], so bit 15 of each half
//    is the comparison result and no carry ever crosses a half.
//  * Compaction: per-thread popcount, a CTA scan in 16x16-cell order, one
//    counter reservation (atomicAdd on the frame's edge counter) per tile,
//    whose round trip is hidden by writing each tile's edges one iteration
//    late.  The cell order makes every 32 consecutive list entries spatially
//    compact: the voting kernel's warps then hit few, consecutive rho bins
//    (distinct shared-memory banks; same-bin lanes merge in ATOMS.POPC.INC).
#include <cstdlib>

#include "ld_internal.cuh"

namespace ld {

// One staged input row, as packed 16-bit pair sums P(x) = r[x] + r[x+1] of the
// chunk's pixels 4k..4k+3 (k = word index):
//   PE[k]  = (P(4k),   P(4k+2))
//   PO[k]  = (P(4k+1), P(4k+3))
//   POL[k] = (P(4k-1), P(4k+1))
// With them, for an output pixel x with rows u (y-1), m (y), d (y+1):
//   A = P_u(x) - P_d(x-1) + M(x),  B = P_d(x) - P_u(x-1) + M(x),
//   M(x) = m[x+1] - m[x-1] = P_m(x) - P_m(x-1)
// (the identity of the file header regrouped), so each input row costs its
// pair sums once and is reused as u, m and d by three output rows.
struct RowP {
  uint32_t PE[4], PO[4], POL[4];
};

// p points at the chunk's first byte in a staged shared-memory row.
__device__ __forceinline__ void load_row(const uint8_t *p, RowP &r) {
  const uint4 w = *reinterpret_cast<const uint4 *>(p);
  const uint32_t wl = *reinterpret_cast<const uint32_t *>(p - 4);
  const uint32_t wr = *reinterpret_cast<const uint32_t *>(p + 16);
  const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
  uint32_t E[5], O[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    E[k] = prmt(ww[k], 0u, 0x4240u);  // (r[4k],   r[4k+2])
    O[k] = prmt(ww[k], 0u, 0x4341u);  // (r[4k+1], r[4k+3])
  }
  E[4] = prmt(wr, 0u, 0x4240u);       // (r[16], r[18])
  // hi half of PO[-1] = r[-1] + r[0]
  const uint32_t pom1 = prmt(wl, 0u, 0x4344u) + prmt(ww[0], 0u, 0x4044u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    r.PE[k] = E[k] + O[k];
    r.PO[k] = O[k] + prmt(E[k], E[k + 1], 0x5432u);  // O + (r[4k+2], r[4k+4])
  }
  r.POL[0] = prmt(pom1, r.PO[0], 0x5432u);
#pragma unroll
  for (int k = 1; k < 4; ++k) r.POL[k] = prmt(r.PO[k - 1], r.PO[k], 0x5432u);
}

// One output row of 16 pixels.  k0 = 2^15 - T2 in both halves, k2 = 2 * k0:
// X = A + k0 has bit 15 set iff A >= T2, k2 - X = -A + k0 iff -A >= T2 (each
// half stays in [0, 2^16): no carry crosses halves).  colm has bit 8j+7 of
// word k set for interior pixels 4k+j.  Returns the edge mask with bit (8j+k)
// set for pixel 4k+j; hb[k] receives the per-byte flags (bit 7 of each byte).
__device__ __forceinline__ uint32_t sobel_row(const RowP &u, const RowP &m, const RowP &d,
                                              uint32_t k0, uint32_t k2, const uint32_t colm[4],
                                              uint32_t hb[4]) {
  uint32_t all = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    // even pixels 4k, 4k+2
    const uint32_t mke = m.PE[k] - m.POL[k] + k0;  // M(x) + k0
    const uint32_t xa = u.PE[k] - d.POL[k] + mke;  // A + k0
    const uint32_t xb = d.PE[k] - u.POL[k] + mke;  // B + k0
    const uint32_t fe = (xa | (k2 - xa) | xb | (k2 - xb)) & 0x80008000u;
    // odd pixels 4k+1, 4k+3
    const uint32_t mko = m.PO[k] - m.PE[k] + k0;
    const uint32_t ya = u.PO[k] - d.PE[k] + mko;
    const uint32_t yb = d.PO[k] - u.PE[k] + mko;
    const uint32_t fo = (ya | (k2 - ya) | yb | (k2 - yb)) & 0x80008000u;
    hb[k] = ((fe >> 8) | fo) & colm[k];  // byte j of word k <-> pixel 4k+j
    all |= hb[k] >> (7 - k);
  }
  return all;
}

template <int SR>
__device__ __forceinline__ void write_edges(const SobelParams &p, const uint32_t masks[SR],
                                            int f, int ybase, int xs, uint32_t off) {
  uint32_t *dst = p.edges + static_cast<int64_t>(f) * p.edge_stride + off;
#pragma unroll
  for (int i = 0; i < SR; ++i) {
    uint32_t m = masks[i];
    const uint32_t yy = static_cast<uint32_t>(ybase + i) << 16;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      *dst++ = yy | static_cast<uint32_t>(xs + 4 * (b & 7) + (b >> 3));
    }
  }
}

template <int SR, int STAGES, int MINB>
__global__ void __launch_bounds__(SB_THREADS, MINB)
    sobel_binarize_compact_kernel(const __grid_constant__ CUtensorMap tmap,
                                  const SobelParams p) {
  constexpr int TILE_H = SR * SB_STRIPS;
  constexpr int BOX_H = TILE_H + 2;
  constexpr int STAGE_BYTES = SB_BOX_W * BOX_H;
  static_assert(STAGE_BYTES % 128 == 0, "stage alignment");
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~static_cast<uintptr_t>(127));
  constexpr int NW = SB_THREADS / 32;
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ uint32_t s_cnt[SB_THREADS];        // per-thread counts, in cell order
  __shared__ uint32_t s_excl[2][SB_THREADS];    // exclusive scan inside each warp
  __shared__ uint32_t s_wt[NW];                 // warp totals
  __shared__ uint32_t s_wbase[2][NW];           // exclusive scan of warp totals
  __shared__ uint32_t s_base[2];                // frame-list base of the tile

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int chunk = tid % SB_CHUNKS;
  const int strip = tid / SB_CHUNKS;
  // List order inside a tile: 16x16-pixel cells (2 strips of one chunk), cells
  // row-major.  32 consecutive list entries then span a compact region, so a
  // warp of the voting kernel hits <= ~32 consecutive rho bins per theta.
  const int ord = ((strip >> 1) * SB_CHUNKS + chunk) * 2 + (strip & 1);
  const uint32_t k0 = static_cast<uint32_t>(32768 - p.t2) * 0x00010001u;
  const uint32_t k2 = k0 + k0;

  auto issue = [&](int tile, int stage) {
    const int f = tile / p.tiles_per_frame;
    const int rem = tile - f * p.tiles_per_frame;
    const int ty = rem / p.tiles_x;
    const int tx = rem - ty * p.tiles_x;
    const int y = p.row_begin + ty * TILE_H - 1 - p.ry0;  // tensor row of smem row 0
    const int x = tx * SB_TILE_W - SB_HALO_L;
    mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES);
    tma_load_3d(smem + stage * STAGE_BYTES, &tmap, &full_bar[stage], x, y, f);
  };

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full_bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      const int tile = blockIdx.x + s * gridDim.x;
      if (tile < p.n_tiles) issue(tile, s);
    }
  }

  // previous tile, written one iteration late so that the counter
  // reservation (a global atomic round trip) overlaps the next tile's work
  uint32_t pmask[SR];
#pragma unroll
  for (int i = 0; i < SR; ++i) pmask[i] = 0u;
  int pf = 0, pybase = 0, pxs = 0;
  uint32_t base_reg = 0;  // thread 0: reservation result of the previous tile

  int it = 0;
  for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++it) {
    const int stage = it % STAGES;
    const uint32_t parity = (it / STAGES) & 1;
    const int cb = it & 1, pb = cb ^ 1;
    const int f = tile / p.tiles_per_frame;
    const int rem = tile - f * p.tiles_per_frame;
    const int ty = rem / p.tiles_x;
    const int tx = rem - ty * p.tiles_x;
    const int y0 = p.row_begin + ty * TILE_H;  // first output row of the tile
    const int xs = tx * SB_TILE_W + chunk * 16;   // first column of this thread's chunk

    // interior columns: bit 8j+7 of word k for pixel 4k+j with 1 <= x <= W-2
    uint32_t colm[4];
    {
      const int lo = 1 - xs, hi = p.width - 2 - xs;  // valid j in [lo, hi]
      if (lo <= 0 && hi >= 15) {
#pragma unroll
        for (int k = 0; k < 4; ++k) colm[k] = 0x80808080u;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t b = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int jj = 4 * k + j;
            if (jj >= lo && jj <= hi) b |= 0x80u << (8 * j);
          }
          colm[k] = b;
        }
      }
    }

    mbar_wait(&full_bar[stage], parity);
    const uint8_t *buf = smem + stage * STAGE_BYTES + SB_HALO_L + chunk * 16;

    uint32_t masks[SR];
    const int ybase = y0 + strip * SR;  // output row of masks[0]
    {
      // rows whose output is computed: interior (1 <= y <= H-2) and owned
      const int ylo = ybase < 1 ? 1 : ybase;
      int yhi = p.height - 2 < p.row_end - 1 ? p.height - 2 : p.row_end - 1;
      RowP r0, r1, r2;
      load_row(buf + (strip * SR + 0) * SB_BOX_W, r0);
      load_row(buf + (strip * SR + 1) * SB_BOX_W, r1);
#pragma unroll
      for (int i = 0; i < SR; ++i) {
        load_row(buf + (strip * SR + i + 2) * SB_BOX_W, r2);
        const int y = ybase + i;
        uint32_t hb[4] = {0u, 0u, 0u, 0u};
        uint32_t all = 0;
        if (y >= ylo && y <= yhi) all = sobel_row(r0, r1, r2, k0, k2, colm, hb);
        masks[i] = all;
        if (p.binary != nullptr && y < p.row_end && xs < p.width) {
          uint8_t *dst = p.binary + static_cast<int64_t>(f) * p.bin_frame_stride +
                         static_cast<int64_t>(y - p.row_begin) * p.bin_pitch + xs;
          // sign-replicating byte permute: 0xFF where bit 7 of the byte is set
          *reinterpret_cast<uint4 *>(dst) =
              make_uint4(prmt(hb[0], 0u, 0xBA98u), prmt(hb[1], 0u, 0xBA98u),
                         prmt(hb[2], 0u, 0xBA98u), prmt(hb[3], 0u, 0xBA98u));
        }
        r0 = r1;
        r1 = r2;
      }
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < SR; ++i) cnt += __popc(masks[i]);
    s_cnt[ord] = cnt;
    if (tid == 0 && it > 0) s_base[pb] = base_reg;
    __syncthreads();  // (A): stage consumed, counts and previous base visible
    if (tid == 0) {
      const int next = tile + STAGES * gridDim.x;
      if (next < p.n_tiles) issue(next, stage);
    }
    if (it > 0 && p.edges != nullptr) {
      const uint32_t off = s_base[pb] + s_wbase[pb][ord >> 5] + s_excl[pb][ord];
      write_edges<SR>(p, pmask, pf, pybase, pxs, off);
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
    for (int i = 0; i < SR; ++i) pmask[i] = masks[i];
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
      write_edges<SR>(p, pmask, pf, pybase, pxs, off);
    }
  }
}

template <int SR, int STAGES, int MINB>
static cudaError_t launch_cfg(const CUtensorMap &tmap, const SobelParams &p, int n_ctas,
                              cudaStream_t stream) {
  auto kern = sobel_binarize_compact_kernel<SR, STAGES, MINB>;
  const size_t smem = static_cast<size_t>(STAGES) * SB_BOX_W * (SR * SB_STRIPS + 2) + 128;
  static bool attr_done[64];  // idempotent per-device attribute; benign race
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_done[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr_done[dev & 63] = true;
  }
  kern<<<n_ctas, SB_THREADS, smem, stream>>>(tmap, p);
  note_launch();
  return cudaGetLastError();
}

SobelCfg sobel_cfg() {
  const char *env = getenv("LD_SOBEL_CFG");
  if (env && env[0] == '4') return SobelCfg{4, 4, 3};
  return SobelCfg{8, 3, 2};
}

cudaError_t launch_sobel(const CUtensorMap &tmap, const SobelParams &p, int sm_count,
                         cudaStream_t stream) {
  const SobelCfg c = sobel_cfg();
  const int64_t max_ctas = static_cast<int64_t>(sm_count) * c.ctas_per_sm;
  const int n_ctas = static_cast<int>(p.n_tiles < max_ctas ? p.n_tiles : max_ctas);
  if (c.sr == 4) return launch_cfg<4, 4, 3>(tmap, p, n_ctas, stream);
  return launch_cfg<8, 3, 2>(tmap, p, n_ctas, stream);
}

}  // namespace ld
