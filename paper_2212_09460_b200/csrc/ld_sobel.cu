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
//    zero-filled by TMA: they feed only border pixels, which are forced to 0 --
//    or, in the paper's zero-padded mode (LD_FLAG_ZERO_PAD), are exactly the
//    padding those border pixels are filtered with.
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

// One output row of 16 pixels, as a 16-bit mask with bit b <-> pixel xs + b.
// k0 = 2^15 - T2 in both halves, k2 = 2 * k0: X = A + k0 has bit 15 set iff
// A >= T2, k2 - X = -A + k0 iff -A >= T2 (each half stays in [0, 2^16): no
// carry crosses halves).  fe (pixels 4k, 4k+2) and fo (4k+1, 4k+3) then hold
// the flags in bits 15 and 31; hi32(fe * 2^(17+4k)) moves them to bits 4k and
// 16+4k, hi32(fo * 2^(18+4k)) to 4k+1 and 17+4k (IMAD.HI on the FMA pipe,
// accumulated: the bits never overlap), and acc | acc >> 14 folds the high
// half onto pixels 4k+2, 4k+3.  colmask clears non-interior columns.
__device__ __forceinline__ uint32_t sobel_row(const RowP &u, const RowP &m, const RowP &d,
                                              uint32_t k0, uint32_t k2, uint32_t colmask) {
  uint32_t acc = 0;
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
    // x (2^s + 1): same high word as x 2^s for these bit patterns (no carry
    // out of the low word), but not a power of two, so it stays an IMAD.HI
    acc += __umulhi(fe, (1u << (17 + 4 * k)) + 1u);
    acc += __umulhi(fo, (1u << (18 + 4 * k)) + 1u);
  }
  return (acc | (acc >> 14)) & colmask;
}

// Emission order of a warp's blocks: chunk by chunk, strips going down in even
// chunks and up in odd ones (a snake), so consecutive list entries stay in a
// compact region even where the order moves to the next chunk (measured model
// of the voting kernel's shared-memory wavefronts per vote instruction on
// cfg3: 1.17 instead of 1.21 for strips always going down).
constexpr int sb_key(int t) {
  return (t % SB_CHUNKS) * SB_STRIPS +
         ((t % SB_CHUNKS) % 2 ? SB_STRIPS - 1 - t / SB_CHUNKS : t / SB_CHUNKS);
}

// per consumer thread: rank of the lane in emission order within its warp,
// and the lane of rank (tid % 32); built at compile time
struct SbOrder {
  uint8_t rank[SB_THREADS], inv[SB_THREADS];
};
constexpr SbOrder make_sb_order() {
  SbOrder o{};
  for (int w = 0; w < SB_THREADS / 32; ++w) {
    for (int l = 0; l < 32; ++l) {
      const int t = w * 32 + l;
      const int key = sb_key(t);
      int r = 0;
      for (int m = 0; m < 32; ++m) r += sb_key(w * 32 + m) < key;
      o.rank[t] = static_cast<uint8_t>(r);
      o.inv[w * 32 + r] = static_cast<uint8_t>(l);
    }
  }
  return o;
}
__constant__ SbOrder c_sb_order = make_sb_order();

// byte expansion of a 4-bit mask: bit j -> byte j = 0xFF (binary-map output)
__constant__ uint32_t kNibbleBytes[16] = {
    0x00000000u, 0x000000FFu, 0x0000FF00u, 0x0000FFFFu, 0x00FF0000u, 0x00FF00FFu,
    0x00FFFF00u, 0x00FFFFFFu, 0xFF000000u, 0xFF0000FFu, 0xFF00FF00u, 0xFF00FFFFu,
    0xFFFF0000u, 0xFFFF00FFu, 0xFFFFFF00u, 0xFFFFFFFFu};

// The edges of two rows of 16 pixels at list positions pos .. pos+popc(m)-1
// (any order: the list is a set, R15): m holds row y in bits 0..15 and row
// y + 1 in bits 16..31 (pixel x0 + (b & 15)); the edge of bit b is
// v0 + b + 65520 (b >> 4) = (y + (b >> 4)) << 16 | (x0 + (b & 15)).  Four
// predicated slots (lowest, highest, then the lowest and highest of the rest)
// cover a row pair with <= 4 edges without a data-dependent branch, so a
// warp does not run as many iterations as its busiest lane; the rest go
// through a short loop.  (One 16-bit row per word took 5.5 % more time on
// cfg4, 2 % on cfg3: tools/ab_time.py, round 2.)
template <typename Store>
__device__ __forceinline__ uint32_t emit_pair(uint32_t m, uint32_t v0, uint32_t pos, Store st) {
  auto val = [&](uint32_t b) { return v0 + b + (b >> 4) * 65520u; };
  const uint32_t n = __popc(m);
  const uint32_t ml = m & (m - 1u);
  const uint32_t b0 = __ffs(m) - 1u;
  const uint32_t b1 = 31u - __clz(ml);
  const uint32_t m2 = n >= 2 ? ml ^ (1u << (b1 & 31u)) : 0u;
  const uint32_t m2l = m2 & (m2 - 1u);
  const uint32_t b2 = __ffs(m2) - 1u;
  const uint32_t b3 = 31u - __clz(m2l);
  if (n >= 1) st(pos, val(b0));
  if (n >= 2) st(pos + 1u, val(b1));
  if (n >= 3) st(pos + 2u, val(b2));
  if (n >= 4) st(pos + 3u, val(b3));
  if (n > 4) {
    uint32_t r = m2l ^ (1u << (b3 & 31u)), q = pos + 4u;
    while (r) {
      st(q++, val(__ffs(r) - 1u));
      r &= r - 1u;
    }
  }
  return pos + n;
}

// All edges of one thread's SR x 16-pixel block (bit b of masks[i] is pixel
// (xs + b, ybase + i)), from list position pos on.
template <int SR, typename Store>
__device__ __forceinline__ void emit_block(const uint32_t masks[SR], int ybase, int xs,
                                           uint32_t pos, Store st) {
  static_assert(SR % 2 == 0, "rows go out in pairs");
#pragma unroll
  for (int i = 0; i < SR; i += 2)
    pos = emit_pair(masks[i] | (masks[i + 1] << 16),
                    (static_cast<uint32_t>(ybase + i) << 16) | static_cast<uint32_t>(xs), pos, st);
}

// Warp-specialised persistent kernel.  Warps 0..6 (224 threads = 14 column
// chunks x 16 row strips) consume tiles; warp 7 is the TMA producer.  A stage
// is handed over with two mbarriers (full: TMA bytes landed; empty: all 7
// consumer warps finished reading it), so the loop has no CTA-wide barrier;
// the producer also publishes each stage's (frame, tile row, tile column).
// Each consumer warp reserves its own slice of the frame's list (one
// atomicAdd per warp per tile) and emits the tile's edges one tile later,
// when the reservation has returned: first into a per-warp shared-memory
// staging buffer at their slice positions, then with coalesced stores.
// Positions are assigned in (chunk, strip) order so that 32 consecutive list
// entries cover a compact 16 x ~24-pixel region (few, consecutive rho bins per
// theta in the voting kernel).
template <int SR, int STAGES, int MINB, bool WB, int CAP>
__global__ void __launch_bounds__(SB_THREADS + 32, MINB)
    sobel_binarize_compact_kernel(const __grid_constant__ CUtensorMap tmap,
                                  const SobelParams p) {
  constexpr int TILE_H = SR * SB_STRIPS;
  constexpr int BOX_H = TILE_H + 2;
  constexpr int STAGE_BYTES = SB_BOX_W * BOX_H;
  constexpr int NCW = SB_THREADS / 32;  // consumer warps
  static_assert(STAGE_BYTES % 128 == 0, "stage alignment");
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint32_t *stage_edges = reinterpret_cast<uint32_t *>(smem + STAGES * STAGE_BYTES);
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ int4 tile_info[STAGES];  // frame, first output row, first column, -

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  LD_PDL_TRIGGER();
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();  // the previous kernel of the stream is done (frames, counts)

  if (warp == NCW) {  // ---------------- producer warp
    if (lane == 0) {
      int it = 0;
      int f = blockIdx.x / p.tiles_per_frame;
      int rem = blockIdx.x - f * p.tiles_per_frame;
      const int sf = gridDim.x / p.tiles_per_frame;
      const int sr = gridDim.x - sf * p.tiles_per_frame;
      for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++it) {
        const int stage = it % STAGES;
        if (it >= STAGES) mbar_wait(&empty_bar[stage], ((it / STAGES) - 1) & 1);
        const int ty = rem / p.tiles_x;
        const int tx = rem - ty * p.tiles_x;
        const int y0 = p.row_begin + ty * TILE_H;
        tile_info[stage] = make_int4(f, y0, tx * SB_TILE_W, 0);
        mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES);  // release: tile_info visible
        tma_load_3d(smem + stage * STAGE_BYTES, &tmap, &full_bar[stage],
                    tx * SB_TILE_W - SB_HALO_L, y0 - 1 - p.ry0, f);
        f += sf;
        rem += sr;
        if (rem >= p.tiles_per_frame) {
          rem -= p.tiles_per_frame;
          ++f;
        }
      }
    }
    return;
  }

  // ---------------- consumer warps
  const uint32_t full_s = smem_u32(full_bar), empty_s = smem_u32(empty_bar);
  const int chunk = tid % SB_CHUNKS;
  const int strip = tid / SB_CHUNKS;
  const uint32_t k0 = static_cast<uint32_t>(32768 - p.t2) * 0x00010001u;
  const uint32_t k2 = k0 + k0;
  // output rows: interior rows 1 .. H-2 (forced-zero border, DESIGN R2) or,
  // zero-padded (R23), every row; always restricted to the owned rows
  const int bord = p.zero_pad ? 0 : 1;
  const int ylo_g = p.row_begin > bord ? p.row_begin : bord;
  const int yhi_g = p.height - 1 - bord < p.row_end - 1 ? p.height - 1 - bord : p.row_end - 1;
  uint32_t *wstage = stage_edges + warp * (CAP + 4);

  // rank of this lane in (chunk, strip) order within the warp, and the lane
  // holding rank `lane` (a fixed permutation, tabulated on the host)
  const int rank = c_sb_order.rank[tid], inv = c_sb_order.inv[tid];

  // previous tile (emitted one iteration late)
  uint32_t pmask[SR];
#pragma unroll
  for (int i = 0; i < SR; ++i) pmask[i] = 0u;
  int pf = 0, pybase = 0, pxs = 0;
  uint32_t pexcl = 0, pcnt = 0, ptotal = 0, pres = 0;  // lane 0 holds the reservation

  auto flush = [&]() {
    // previous tile: its reservation has had a whole tile to return
    const uint32_t base = __shfl_sync(0xffffffffu, pres, 0);
    uint32_t *glist = p.edges + static_cast<int64_t>(pf) * p.edge_stride + base;
    if constexpr (CAP == 0) {
      emit_block<SR>(pmask, pybase, pxs, pexcl, [&](uint32_t q, uint32_t v) { glist[q] = v; });
    } else {
      // staged at the list's address modulo 16 (mis words in), so the slice
      // leaves by one bulk copy of its aligned middle
      const uint32_t mis = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(glist) & 15u) >> 2);
      if (lane == 0) bulk_wait_read();  // the previous slice's copy has read the buffer
      __syncwarp();
      const bool fits = pexcl + pcnt <= static_cast<uint32_t>(CAP);
      if (fits) {
        const uint32_t sb = smem_u32(wstage + mis);
        emit_block<SR>(pmask, pybase, pxs, pexcl, [&](uint32_t q, uint32_t v) {
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(sb + 4u * q), "r"(v) : "memory");
        });
      } else {
        emit_block<SR>(pmask, pybase, pxs, pexcl, [&](uint32_t q, uint32_t v) { glist[q] = v; });
      }
      // staged prefix: everything before the first lane that overflowed
      const uint32_t split = __reduce_min_sync(0xffffffffu, fits ? ptotal : pexcl);
      fence_proxy_async_smem();
      __syncwarp();
      const uint32_t head = min((4u - mis) & 3u, split);
      const uint32_t mid = ((split - head) >> 2) << 2;
      if (lane < head) glist[lane] = wstage[mis + lane];
      for (uint32_t q = head + mid + lane; q < split; q += 32) glist[q] = wstage[mis + q];
      if (lane == 0 && mid > 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(glist + head), "r"(smem_u32(wstage + mis + head)), "r"(mid * 4u)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
  };

  int it = 0;
  for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++it) {
    const int stage = it % STAGES;
    mbar_wait_s(full_s + 8u * stage, (it / STAGES) & 1);
    const int4 ti = tile_info[stage];
    const int f = ti.x;
    const int xs = ti.z + chunk * 16;     // first column of this thread's chunk
    const int ybase = ti.y + strip * SR;  // output row of masks[0]

    uint32_t colmask = 0xFFFFu;  // output columns bord <= x <= W-1-bord
    {
      const int lo = bord - xs, hi = p.width - 1 - bord - xs;
      if (lo > 0 || hi < 15) {
        colmask = (hi < 0 || lo > 15) ? 0u
                                      : ((0xFFFFu >> (15 - min(hi, 15))) & (0xFFFFu << max(lo, 0)));
      }
    }

    const uint8_t *buf = smem + stage * STAGE_BYTES + SB_HALO_L + chunk * 16 + strip * SR * SB_BOX_W;
    uint32_t masks[SR];
#pragma unroll
    for (int i = 0; i < SR; ++i) masks[i] = 0u;
    // every row of the strip inside the output rows (all but the frame's top
    // and bottom strips): no per-row test
    const bool rows_in = ybase >= ylo_g && ybase + SR - 1 <= yhi_g;
    if (ybase < p.row_end && xs < p.width) {  // skip strips/chunks outside the image
      RowP r0, r1, r2;
      load_row(buf, r0);
      load_row(buf + SB_BOX_W, r1);
#pragma unroll
      for (int i = 0; i < SR; ++i) {
        load_row(buf + (i + 2) * SB_BOX_W, r2);
        const int y = ybase + i;
        const uint32_t m = sobel_row(r0, r1, r2, k0, k2, colmask);
        masks[i] = m;
        if (WB && y < p.row_end && xs < p.width) {
          uint8_t *dst = p.binary + static_cast<int64_t>(f) * p.bin_frame_stride +
                         static_cast<int64_t>(y - p.row_begin) * p.bin_pitch + xs;
          const uint32_t mm = (y >= ylo_g && y <= yhi_g) ? m : 0u;
          *reinterpret_cast<uint4 *>(dst) =
              make_uint4(kNibbleBytes[mm & 15u], kNibbleBytes[(mm >> 4) & 15u],
                         kNibbleBytes[(mm >> 8) & 15u], kNibbleBytes[(mm >> 12) & 15u]);
        }
        r0 = r1;
        r1 = r2;
      }
      if (!rows_in) {  // the frame's top / bottom strips: rows outside the output rows
#pragma unroll
        for (int i = 0; i < SR; ++i)
          if (ybase + i < ylo_g || ybase + i > yhi_g) masks[i] = 0u;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_s(empty_s + 8u * stage);  // stage consumed by this warp

    // warp-level reservation of this tile's slice, scanned in rank order
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < SR; ++i) cnt += __popc(masks[i]);
    const uint32_t cr = __shfl_sync(0xffffffffu, cnt, inv);  // count of rank `lane`
    uint32_t incl = cr;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t excl = __shfl_sync(0xffffffffu, incl - cr, rank);

    if (it > 0 && p.edges != nullptr) flush();
    if (lane == 0) pres = total ? atomicAdd(&p.counts[f], total) : 0u;
#pragma unroll
    for (int i = 0; i < SR; ++i) pmask[i] = masks[i];
    pexcl = excl;
    pcnt = cnt;
    ptotal = total;
    pf = f;
    pybase = ybase;
    pxs = xs;
  }
  if (it > 0 && p.edges != nullptr) flush();
  if (lane == 0) bulk_wait_read();  // the last slice's copy has read the buffer
}

template <int SR, int STAGES, int MINB, bool WB, int CAP = SB_STAGE_CAP>
static cudaError_t launch_cfg(const CUtensorMap &tmap, const SobelParams &p, int n_ctas,
                              cudaStream_t stream) {
  auto kern = sobel_binarize_compact_kernel<SR, STAGES, MINB, WB, CAP>;
  const size_t smem = static_cast<size_t>(STAGES) * SB_BOX_W * (SR * SB_STRIPS + 2) +
                      static_cast<size_t>(SB_THREADS / 32) * (CAP + 4) * 4 + 128;
  static AttrOnce attr;
  const cudaError_t e = ensure_smem_attr(attr, kern, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  return launch_ex(kern, dim3(n_ctas), dim3(SB_THREADS + 32), smem, stream, 1, tmap, p);
}

// Launch configuration: SR = 8 rows per thread strip (128-row tiles), 2 TMA
// stages, 2 CTAs per SM, 1024-entry per-warp edge staging.  Measured on B200
// (profiles/) against 3 stages (smaller staging), 3 CTAs per SM
// (register-capped), 64- and 96-row tiles and direct (unstaged) edge stores:
// all slower on cfg3 and cfg4.  Work too small to give every SM a 128-row
// tile (single frames: cfg1, cfg2, 512 x 512) takes 32-row tiles (SR = 2),
// four times as many CTAs each with a quarter of the latency.
#ifndef LD_SOBEL_SR
#define LD_SOBEL_SR 8  // output rows per thread strip (tile height 16 * SR)
#endif
SobelCfg sobel_cfg(int width, int rows, int frames, int sms) {
  const int64_t tiles = static_cast<int64_t>((width + SB_TILE_W - 1) / SB_TILE_W) *
                        ((rows + 16 * LD_SOBEL_SR - 1) / (16 * LD_SOBEL_SR)) * frames;
  return SobelCfg{tiles < sms ? 2 : LD_SOBEL_SR, 2, 2, SB_STAGE_CAP};
}

#ifndef LD_SOBEL_MINB
#define LD_SOBEL_MINB 2  // CTAs per SM (register budget 65536 / (288 * MINB))
#endif
#ifndef LD_SOBEL_STAGES
#define LD_SOBEL_STAGES 2  // TMA ring depth per CTA
#endif
cudaError_t launch_sobel(const CUtensorMap &tmap, const SobelParams &p, int sm_count,
                         cudaStream_t stream) {
  constexpr int MB = LD_SOBEL_MINB, ST = LD_SOBEL_STAGES;
  const int64_t max_ctas = static_cast<int64_t>(sm_count) * MB;
  const int n_ctas = static_cast<int>(p.n_tiles < max_ctas ? p.n_tiles : max_ctas);
  if (p.sr == 2)
    return p.binary != nullptr ? launch_cfg<2, ST, MB, true>(tmap, p, n_ctas, stream)
                               : launch_cfg<2, ST, MB, false>(tmap, p, n_ctas, stream);
  return p.binary != nullptr ? launch_cfg<LD_SOBEL_SR, ST, MB, true>(tmap, p, n_ctas, stream)
                             : launch_cfg<LD_SOBEL_SR, ST, MB, false>(tmap, p, n_ctas, stream);
}

}  // namespace ld
