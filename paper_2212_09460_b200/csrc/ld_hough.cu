// ld_hough.cu -- B3: theta-partitioned shared-memory Hough voting, sm_100a;
//                B5: shared-memory atomic microbenchmark (the voting roofline).
//
// Paper: Eq. 3, voting, 180 one-degree PEs, the GPU
// design of one thread block per theta with the voting space in block shared
// memory and atomic adds for colliding votes; the half-angle
// symmetry of Eq. 4-5.  DESIGN.md 6.2.
//
// Design: the paper gives each theta its own 48 KB block (K80).  On sm_100a a
// CTA owns a BAND of theta rows -- as many rows of n_rho uint32 counters as fit
// in half of the 227 KB opt-in shared memory (two CTAs per SM, so one CTA's
// prologue and write-out overlap the other's voting) -- and each frame's edge
// list is streamed n_theta / rows times instead of n_theta times.  For every
// row of the band a lane issues one red.shared.add.u32 per edge at
// ((x*C + y*S + 2^14 + (D << 15)) >> 15) (SASS: ATOMS.POPC.INC; lanes that
// hit the same counter merge in hardware).  The host range proof (ld_api.cu)
// makes a per-vote bounds check unnecessary.  The band leaves shared memory
// by bulk (TMA engine) copies: no global atomics anywhere.
//
// Measured cost model of ATOMS on B200 (tools/atoms_probe.cu,
// profiles/r02_atoms_probe.md): one wavefront per clock per SM; lanes on the
// same address merge for free; k distinct addresses in one bank cost k
// wavefronts.  So a warp's 32 votes cost one wavefront iff their rho bins span
// fewer than 32 consecutive counters -- which is why ld_sobel.cu emits edges
// in a spatially compact order.
//
// While a band is in shared memory the kernel also writes, for the peak
// search (DESIGN R25, R30), (a) per warp the largest count it saw and its
// cell, and (b) the maximum of every 1 KB chunk of the accumulator.
#include <cooperative_groups.h>
#include <cstdlib>

#include "ld_internal.cuh"

namespace ld {

#ifndef LD_HV_UNROLL
#define LD_HV_UNROLL 4  // band rows per unrolled step (plain kernel)
#endif
#ifndef LD_HV_CTAS_MAX
#define LD_HV_CTAS_MAX 2  // experiment: 1 = always one CTA per SM (taller bands)
#endif
#ifndef LD_HV_PAIR_UNROLL
#define LD_HV_PAIR_UNROLL 2  // pairs per unrolled step (paired kernel)
#endif

// ---------------------------------------------------------------------------
// Shared pieces
// ---------------------------------------------------------------------------

// dst[0 .. ncell) = src[0 .. ncell), src and dst congruent modulo 16 bytes:
// the aligned middle by one bulk shared->global copy (issued by thread 0 and
// committed as a bulk group; the caller waits for it before the CTA exits),
// the <= 3 head and tail words by plain stores.  The caller must have made
// the shared-memory writes visible to the async proxy (fence.proxy.async by
// every writing thread, then a barrier).
__device__ __forceinline__ void bulk_rows_out(uint32_t *dst, const uint32_t *src, int ncell,
                                              int tid, int nt) {
  if (ncell <= 0) return;
  const int mis = static_cast<int>((reinterpret_cast<uintptr_t>(dst) & 15u) >> 2);
  const int head = min((4 - mis) & 3, ncell);
  const int mid = ((ncell - head) >> 2) << 2;
  if (tid < head) dst[tid] = src[tid];
  for (int i = head + mid + tid; i < ncell; i += nt) dst[i] = src[i];
  if (tid == 0 && mid > 0) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + head),
                 "r"(smem_u32(src + head)), "r"(static_cast<uint32_t>(mid) * 4u)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}

// Running per-warp best of the summaries: the largest chunk maximum seen and
// the chunk (its shared-memory words and their global address).  Chunks are
// visited in increasing address order per warp, so the strict '>' keeps the
// first (lowest-address) chunk among equal maxima.
struct SegBest {
  uint32_t v = 0;
  const uint32_t *sm = nullptr;  // shared-memory copy of the chunk's first word
  const uint32_t *gl = nullptr;  // its global address
};

// Summaries of one block of counters on its way out: dst[0 .. ncell) in
// global memory, src the shared-memory copy (congruent modulo 16 bytes).  The
// accumulator is cut into SEG_BYTES-aligned chunks of GLOBAL memory (DESIGN
// R30); the maximum of the block's counters in each chunk goes to
// segmax[chunk - first chunk of the frame]: a plain store for a chunk wholly
// inside the block, an atomicMax for a chunk the block shares with a
// neighbouring block or frame (at most two per block; the host zeroes segmax
// before the launch).  Warp `wi` of `nw` takes chunks wi, wi+nw, ...: two
// 16-byte shared loads per lane (256 words = 32 lanes x 8), a max tree and
// one REDUX.MAX.
__device__ __forceinline__ void summarize_block(const uint32_t *dst, const uint32_t *src,
                                                int ncell, uintptr_t frame_chunk0,
                                                uint32_t *segmax_frame, int wi, int nw, int lane,
                                                SegBest &best) {
  if (ncell <= 0) return;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(dst);
  const uintptr_t a1 = reinterpret_cast<uintptr_t>(dst + ncell);
  const uintptr_t q0 = a0 / SEG_BYTES, q1 = (a1 - 1) / SEG_BYTES;
  for (uintptr_t q = q0 + wi; q <= q1; q += nw) {
    const uintptr_t c0 = q * SEG_BYTES;
    if (c0 >= a0 && c0 + SEG_BYTES <= a1) {
      const uint32_t *sc = src + (c0 - a0) / 4;  // 16-byte aligned (congruent copies)
      const uint4 u = reinterpret_cast<const uint4 *>(sc)[lane];
      const uint4 w = reinterpret_cast<const uint4 *>(sc)[32 + lane];
      const uint32_t v = max(max(max(u.x, u.y), max(u.z, u.w)), max(max(w.x, w.y), max(w.z, w.w)));
      const uint32_t m = __reduce_max_sync(0xffffffffu, v);
      if (m > best.v) {
        best.v = m;
        best.sm = sc;
        best.gl = reinterpret_cast<const uint32_t *>(c0);
      }
      if (lane == 0) segmax_frame[q - frame_chunk0] = m;
    } else {  // the block's part of a shared chunk, word by word
      uint32_t v = 0u;
      for (int i = lane; i < SEG_BYTES / 4; i += 32) {
        const uintptr_t a = c0 + 4u * i;
        if (a >= a0 && a < a1) v = max(v, src[(a - a0) / 4]);
      }
      const uint32_t m = __reduce_max_sync(0xffffffffu, v);
      if (lane == 0 && m) atomicMax(segmax_frame + (q - frame_chunk0), m);
    }
  }
}

// The warp's hint key (value << 32 | ~cell index) from its best chunk: the
// first word holding the maximum.  0 when the warp saw only zeros.
__device__ __forceinline__ unsigned long long seg_best_key(const SegBest &b,
                                                           const uint32_t *frame, int lane) {
  if (b.v == 0u) return 0ull;
  // lane l's words: 4l .. 4l+3 and 128+4l .. 128+4l+3
  const uint4 u = reinterpret_cast<const uint4 *>(b.sm)[lane];
  const uint4 w = reinterpret_cast<const uint4 *>(b.sm)[32 + lane];
  const int lo = u.x == b.v ? 0 : u.y == b.v ? 1 : u.z == b.v ? 2 : u.w == b.v ? 3 : 99;
  const int hi = w.x == b.v ? 0 : w.y == b.v ? 1 : w.z == b.v ? 2 : w.w == b.v ? 3 : 99;
  const uint32_t bl = __ballot_sync(0xffffffffu, lo < 99), bh = __ballot_sync(0xffffffffu, hi < 99);
  const int src_lane = bl ? __ffs(bl) - 1 : __ffs(bh) - 1;
  const int sub = __shfl_sync(0xffffffffu, bl ? lo : hi, src_lane);
  const int word = (bl ? 0 : 128) + 4 * src_lane + sub;
  const uint32_t idx = static_cast<uint32_t>((b.gl + word) - frame);
  return (static_cast<unsigned long long>(b.v) << 32) | (0xFFFFFFFFu - idx);
}

__device__ __forceinline__ void write_hint_header(const HoughParams &p, int nwarps) {
  uint32_t *h = p.hint_hdr;
  h[0] = HINT_MAGIC;
  h[1] = static_cast<uint32_t>(p.batch);
  h[2] = static_cast<uint32_t>(p.n_theta);
  h[3] = static_cast<uint32_t>(p.n_rho);
  h[4] = static_cast<uint32_t>(p.n_bands);
  h[5] = static_cast<uint32_t>(nwarps);
  h[6] = static_cast<uint32_t>(p.n_seg);
  const uint64_t a = reinterpret_cast<uintptr_t>(p.acc);  // segmax is tied to this address
  h[7] = static_cast<uint32_t>(a);
  h[8] = static_cast<uint32_t>(a >> 32);
}

// ---------------------------------------------------------------------------
// Plain kernel (any table): one block of rows t0 .. t0+nr-1 per CTA
// ---------------------------------------------------------------------------

// One block of 32 x EPL consecutive list entries of a warp (entry
// blk + 32j + lane in lane `lane`), voted into every row of the band.
// Entries past `end` (FULL = false) vote into the scratch word instead of
// being branched around: no divergent control flow in the tail.
template <int EPL, bool FULL>
__device__ __forceinline__ void vote_block(const uint32_t *el, uint32_t blk, uint32_t end,
                                           int lane, int nr, const uint4 *rowk,
                                           uint32_t scratch) {
  uint32_t xs[EPL], ys[EPL];
  bool ok[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    const uint32_t e = blk + 32u * j + lane;
    ok[j] = FULL || e < end;
    const uint32_t q = ok[j] ? __ldg(el + e) : 0u;
    xs[j] = q & 0xFFFFu;
    ys[j] = q >> 16;
  }
  constexpr int HV_UNROLL = LD_HV_UNROLL;
#pragma unroll HV_UNROLL
  for (int r = 0; r < nr; ++r) {
    const uint4 k = rowk[r];
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const uint32_t a = ((xs[j] * k.x + ys[j] * k.y + k.z) >> 13) & ~3u;
      red_shared_add(FULL || ok[j] ? a : scratch, 1u);
    }
  }
}

template <int CTAS>
__global__ void __launch_bounds__(HV_THREADS / CTAS, CTAS)
    hough_vote_kernel(const HoughParams p, const __grid_constant__ TrigTable trig) {
  constexpr int NT = HV_THREADS / CTAS;
  constexpr int NWARPS = NT / 32;
  extern __shared__ __align__(16) uint32_t slice_raw[];
  __shared__ uint4 rowk[HV_MAX_ROWS];  // per row: C, S, K = koff + (row address << 13)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int band = blockIdx.x;
  const int f = blockIdx.y;
  const int t0 = band * p.rows_per_band;
  const int nr = min(p.rows_per_band, p.n_theta - t0);
  const int ncell = nr * p.n_rho;
  uint32_t *dst = p.acc + (static_cast<int64_t>(f) * p.n_theta + t0) * p.n_rho;
  // The slice starts at the same address modulo 16 as its destination, so the
  // write-out can be one bulk copy of its 16-byte-aligned middle part.
  const int mw = static_cast<int>((reinterpret_cast<uintptr_t>(dst) & 15u) >> 2);
  uint32_t *slice = slice_raw + mw;
  const uint32_t sbase = smem_u32(slice);
  const uint32_t row_bytes = static_cast<uint32_t>(p.n_rho) * 4u;

  {
    uint4 *s4 = reinterpret_cast<uint4 *>(slice_raw);
    const int n4 = (mw + ncell + 1 + 3) >> 2;
    for (int i = tid; i < n4; i += NT) s4[i] = make_uint4(0u, 0u, 0u, 0u);
    // The byte address of the counter of (row r, bin rho) is
    //   sbase + r*row_bytes + 4*rho = ((v + ((sbase + r*row_bytes) << 13)) >> 13) & ~3
    // with v = x*C + y*S + koff in [0, 2^31) (host range proof) and the row
    // address < 2^18, so the folded sum stays below 2^32: exact in uint32.
    for (int i = tid; i < nr; i += NT)
      rowk[i] = make_uint4(static_cast<uint32_t>(trig.c[t0 + i]), static_cast<uint32_t>(trig.s[t0 + i]),
                           static_cast<uint32_t>(p.koff) + ((sbase + i * row_bytes) << 13), 0u);
  }
  __syncthreads();

  const uint32_t n_edges = p.counts[f];
  const uint32_t *el = p.edges + static_cast<int64_t>(f) * p.edge_stride;

  // Warps take blocks of consecutive list entries, interleaved across the
  // CTA's warps: 16 entries per lane while whole rounds of such blocks remain
  // (fewer edge loads per vote), then 8 per lane, then a predicated tail, so
  // the warps finish within one short block of each other.
  uint32_t base = 0;
  const uint32_t scratch = smem_u32(slice + ncell);  // inside the allocation, never written out
  for (; base + NWARPS * 32u * 16u <= n_edges; base += NWARPS * 32u * 16u)
    vote_block<16, true>(el, base + warp * 32u * 16u, n_edges, lane, nr, rowk, scratch);
  uint32_t blk = base + static_cast<uint32_t>(warp) * (32u * 8u);
  for (; blk + 32u * 8u <= n_edges; blk += NWARPS * 32u * 8u)
    vote_block<8, true>(el, blk, n_edges, lane, nr, rowk, scratch);
  if (blk < n_edges) vote_block<8, false>(el, blk, n_edges, lane, nr, rowk, scratch);
  fence_proxy_async_smem();
  __syncthreads();

  bulk_rows_out(dst, slice, ncell, tid, NT);
  if (p.hint_keys) {
    SegBest best;
    const uint32_t *frame = p.acc + static_cast<int64_t>(f) * p.n_theta * p.n_rho;
    summarize_block(dst, slice, ncell, reinterpret_cast<uintptr_t>(frame) / SEG_BYTES,
                    p.segmax + static_cast<int64_t>(f) * p.n_seg, warp, NWARPS, lane, best);
    const unsigned long long key = seg_best_key(best, frame, lane);
    if (lane == 0) p.hint_keys[(static_cast<int64_t>(f) * p.n_bands + band) * NWARPS + warp] = key;
    if (f == 0 && band == 0 && tid == 0) write_hint_header(p, NWARPS);
  }
  if (tid == 0) bulk_wait_read();
}

static int rows_per_band(int n_theta, int n_rho, size_t limit, int *n_bands) {
  const size_t row = static_cast<size_t>(n_rho) * 4u;
  int rows_max = static_cast<int>(limit / row);
  if (rows_max > HV_MAX_ROWS) rows_max = HV_MAX_ROWS;
  if (rows_max < 1) return 0;
  const int nb = (n_theta + rows_max - 1) / rows_max;
  *n_bands = nb;
  return (n_theta + nb - 1) / nb;
}

int hough_plan(int n_theta, int n_rho, size_t smem_optin, int *ctas, int *rpb, int *n_bands,
               size_t *smem_bytes) {
  // per CTA: the slice (+16 bytes of alignment shift, +1 scratch word), rowk, a margin
  const size_t fixed = sizeof(uint4) * HV_MAX_ROWS + 1024 + 32;
  int nb1 = 0, nb2 = 0;
  const int r1 = rows_per_band(n_theta, n_rho, smem_optin - fixed, &nb1);
  if (r1 < 1) return 0;
  const int r2 = rows_per_band(n_theta, n_rho, smem_optin / 2 - fixed, &nb2);
  const bool two = LD_HV_CTAS_MAX > 1 && r2 >= 8 &&
                   (smem_optin - fixed) / (static_cast<size_t>(n_rho) * 4u) >= 16;
  *ctas = two ? 2 : 1;
  *rpb = two ? r2 : r1;
  *n_bands = two ? nb2 : nb1;
  *smem_bytes = ((static_cast<size_t>(*rpb) * n_rho * 4 + 15) / 16) * 16 + 32;
  return 1;
}

static AttrOnce g_hough_attr[3];

cudaError_t launch_hough(const HoughParams &p, const TrigTable &trig, int ctas, size_t smem_bytes,
                         cudaStream_t stream) {
  auto kern = ctas == 2 ? hough_vote_kernel<2> : hough_vote_kernel<1>;
  cudaError_t e = ensure_smem_attr(g_hough_attr[ctas], kern, -(227 * 1024 / ctas));
  if (e != cudaSuccess) return e;
  dim3 grid(p.n_bands, p.batch);
  kern<<<grid, HV_THREADS / ctas, smem_bytes, stream>>>(p, trig);
  note_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Half-angle paired voting (NEXT 2; the paper's Eq. 4-5): for a
// table with C[n-t] = -C[t] and S[n-t] = S[t], the rows t and n - t share
// Q = y*S[t] + K:  V_t = x*C[t] + Q,  V_{n-t} = Q - x*C[t] = V_t - 2x*C[t].
// A CTA holds pairs p0 .. p0+np-1.  Its shared memory has two blocks of np
// rows: block 1 holds rows t = p0 + i at slot i (ascending, like acc); block 2
// holds the partners n - t at slot np-1-i, i.e. rows n-p0-np+1 .. n-p0
// ASCENDING as well -- so each block leaves by ONE bulk copy.  The partner of
// slot i lies delta_i = (block-2 row np-1-i) - (block-1 row i) bytes above it;
// delta_i is warp-uniform per pair, so it folds into the ATOMS address as a
// uniform-register offset ([R+UR]):
//   addr(t)   = ((x*C + Q) >> 13) & ~3              (Q = y*S + koff + (row address << 13))
//   addr(n-t) = ((x*(-2C) + V_t) >> 13) & ~3, + delta_i
// 9 instructions per 2 votes (3 IMAD, 2 SHF, 2 LOP3, 2 ATOMS).  Folding is
// exact as in the plain kernel: V in [0, 2^31) for both rows (host range
// proof, mirrored entries included), addresses < 2^18.
// Pair p = 0 and p = n/2 (n even) have no partner: their mirror votes land in
// a block-2 row that is not written out (row n, and row n/2 a second time).
// ---------------------------------------------------------------------------
int hough_pair_count(int n_theta) { return n_theta / 2 + 1; }

template <int EPL, bool FULL>
__device__ __forceinline__ void vote_block_pairs(const uint32_t *el, uint32_t blk, uint32_t end,
                                                 int lane, int np, const uint4 *rowk,
                                                 uint32_t row_bytes, uint32_t delta0,
                                                 uint32_t scratch, uint32_t win) {
  // one 32-bit load per entry: the kernel is bound by the L1 data pipe
  // (shared-memory atomics + these loads, one wavefront per clock per SM),
  // so the unpacking ALU instructions are cheaper than a second 16-bit load
  const uint32_t *pe = el + blk + lane;
  uint32_t xs[EPL], ys[EPL];
  bool ok[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    ok[j] = FULL || blk + 32u * j + lane < end;
    const uint32_t q = ok[j] ? __ldg(pe + 32 * j) : 0u;
    xs[j] = q & 0xFFFFu;
    ys[j] = q >> 16;
  }
  constexpr int PAIR_UNROLL = LD_HV_PAIR_UNROLL;
#pragma unroll PAIR_UNROLL
  for (int r = 0; r < np; ++r) {
    const uint4 k = rowk[r];  // C, S, K, -2C (one broadcast shared load per pair)
    const uint32_t delta = delta0 - static_cast<uint32_t>(r) * 2u * row_bytes;  // uniform
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const uint32_t v1 = xs[j] * k.x + (ys[j] * k.y + k.z);
      const uint32_t v2 = xs[j] * k.w + v1;
      // shift + mask (the IMAD.HI form 4 * hi32(v * 2^17), on the FMA pipe,
      // measured slower); win = the CTA's shared window (its cluster rank
      // bits), added as a uniform-register offset of the ATOMS
      red_shared_add((FULL || ok[j] ? (v1 >> 13) & ~3u : scratch) + win, 1u);
      red_shared_add((FULL || ok[j] ? (v2 >> 13) & ~3u : scratch - delta) + (delta + win), 1u);
    }
  }
}

// Cluster epilogue (G > 1: a band's edges are split over the G CTAs of a
// thread-block cluster, each voting into its own shared-memory copy of the
// band -- for single frames, whose bands alone would leave most SMs idle,
// DESIGN 6.2).  The copies are summed over distributed shared memory: the
// band's global chunks (SEG_BYTES-aligned, as the summaries) are dealt to the
// cluster's CTAs and their warps; each lane adds the G copies of its words,
// stores the sums and folds them into the chunk maximum (atomicMax: a chunk
// can also belong to a neighbouring band's cluster) and into its best cell
// (the CTA's hint key).
template <int G, int NWARPS>
__device__ __forceinline__ void cluster_reduce_out(const HoughParams &p, uint32_t *dst,
                                                   int smem_off, int ncell,
                                                   uint32_t *const *copies, uintptr_t fc0,
                                                   const uint32_t *frame, int rank, int warp,
                                                   int lane, unsigned long long &best) {
  if (ncell <= 0) return;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(dst);
  const uintptr_t a1 = reinterpret_cast<uintptr_t>(dst + ncell);
  const uintptr_t q0 = a0 / SEG_BYTES, q1 = (a1 - 1) / SEG_BYTES;
  uint32_t *segmax = p.hint_keys ? p.segmax + static_cast<int64_t>(blockIdx.y) * p.n_seg : nullptr;
  for (uintptr_t q = q0 + rank + static_cast<uintptr_t>(G) * warp; q <= q1;
       q += static_cast<uintptr_t>(G) * NWARPS) {
    uint32_t m = 0u;
#pragma unroll
    for (int i = 0; i < SEG_BYTES / 128; ++i) {
      const uintptr_t a = q * SEG_BYTES + 4u * (32u * i + lane);
      if (a >= a0 && a < a1) {
        const int li = static_cast<int>((a - a0) / 4);
        uint32_t v = 0u;
#pragma unroll
        for (int c = 0; c < G; ++c) v += copies[c][smem_off + li];
        dst[li] = v;
        m = max(m, v);
        const unsigned long long key =
            (static_cast<unsigned long long>(v) << 32) |
            (0xFFFFFFFFu - static_cast<uint32_t>((dst + li) - frame));
        if (v && key > best) best = key;
      }
    }
    if (segmax) {
      m = __reduce_max_sync(0xffffffffu, m);
      if (lane == 0 && m) atomicMax(segmax + (q - fc0), m);
    }
  }
}

template <int CTAS, int G>
__global__ void __launch_bounds__(HV_THREADS / CTAS, CTAS)
    hough_vote_pairs_kernel(const HoughParams p, const __grid_constant__ TrigTable trig) {
  constexpr int NT = HV_THREADS / CTAS;
  constexpr int NWARPS = NT / 32;
  extern __shared__ __align__(16) uint32_t slice_raw[];
  __shared__ uint4 rowk[HV_MAX_ROWS];  // per pair: C, S, K = koff + (row t address << 13), -2C

  LD_PDL_TRIGGER();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int band = blockIdx.x / G;
  const int rank = G > 1 ? static_cast<int>(blockIdx.x % G) : 0;  // rank in the cluster
  const int f = blockIdx.y;
  const int n_rho = p.n_rho, n_theta = p.n_theta;
  const int p0 = band * p.rows_per_band;
  const int np = min(p.rows_per_band, p.n_pairs - p0);
  const int ncell = np * n_rho;
  uint32_t *frame = p.acc + static_cast<int64_t>(f) * n_theta * n_rho;
  // block 1: rows p0 .. p0+np-1; block 2: rows g2 .. g2+np-1 with g2 = n-p0-np+1
  const int g2 = n_theta - p0 - np + 1;
  uint32_t *dst1 = frame + static_cast<int64_t>(p0) * n_rho;
  uint32_t *dst2 = frame + static_cast<int64_t>(g2) * n_rho;  // may point one row past acc
  // each block at its destination's address modulo 16 (bulk write-out)
  const int mw1 = static_cast<int>((reinterpret_cast<uintptr_t>(dst1) & 15u) >> 2);
  const int mw2 = static_cast<int>((reinterpret_cast<uintptr_t>(dst2) & 15u) >> 2);
  const int h2 = ((mw1 + ncell + 3) >> 2) << 2;  // block 2's 16-byte-aligned base (words)
  uint32_t *blk1 = slice_raw + mw1;
  uint32_t *blk2 = slice_raw + h2 + mw2;
  const uint32_t row_bytes = static_cast<uint32_t>(n_rho) * 4u;
  // Shared addresses are the CTA's window (bits 24+: its rank in a cluster,
  // 0 otherwise) plus an offset < 2^18; only offsets are folded into K (the
  // << 13 must not overflow 32 bits), the window goes into the ATOMS.
  const uint32_t win = smem_u32(slice_raw) & 0xFF000000u;
  // partner distance of slot i: delta0 - i * 2 row_bytes
  const uint32_t delta0 = smem_u32(blk2) - smem_u32(blk1) + static_cast<uint32_t>(np - 1) * row_bytes;
  const uint32_t scratch = smem_u32(blk2 + ncell) - win;  // inside the allocation, never written out
  {
    uint4 *s4 = reinterpret_cast<uint4 *>(slice_raw);
    const int n4 = (h2 + mw2 + ncell + 1 + 3) >> 2;
    for (int i = tid; i < n4; i += NT) s4[i] = make_uint4(0u, 0u, 0u, 0u);
    const uint32_t sbase = smem_u32(blk1) - win;
    for (int i = tid; i < np; i += NT) {
      const int t = p0 + i;
      rowk[i] = make_uint4(static_cast<uint32_t>(trig.c[t]), static_cast<uint32_t>(trig.s[t]),
                           static_cast<uint32_t>(p.koff) + ((sbase + i * row_bytes) << 13),
                           static_cast<uint32_t>(-2 * trig.c[t]));
    }
  }
  __syncthreads();
  // (the slice zeroed and the trig rows staged while the previous kernel of
  // the stream -- the edge list's producer -- finished)
  pdl_wait();

  // this CTA's part of the frame's list: all of it, or (cluster) the rank-th
  // of G parts, cut at multiples of 32 entries
  const uint32_t n_all = p.counts[f];
  const uint32_t e_lo = G > 1 ? ((n_all / 32u) * rank / G) * 32u : 0u;
  const uint32_t e_hi = G > 1 ? (rank == G - 1 ? n_all : ((n_all / 32u) * (rank + 1) / G) * 32u)
                              : n_all;
  const uint32_t n_edges = e_hi - e_lo;
  const uint32_t *el = p.edges + static_cast<int64_t>(f) * p.edge_stride + e_lo;
  uint32_t base = 0;
  for (; base + NWARPS * 32u * 16u <= n_edges; base += NWARPS * 32u * 16u)
    vote_block_pairs<16, true>(el, base + warp * 32u * 16u, n_edges, lane, np, rowk, row_bytes,
                               delta0, scratch, win);
  uint32_t blk = base + static_cast<uint32_t>(warp) * (32u * 8u);
  for (; blk + 32u * 8u <= n_edges; blk += NWARPS * 32u * 8u)
    vote_block_pairs<8, true>(el, blk, n_edges, lane, np, rowk, row_bytes, delta0, scratch, win);
  if (blk < n_edges)
    vote_block_pairs<8, false>(el, blk, n_edges, lane, np, rowk, row_bytes, delta0, scratch,
                               win);
  fence_proxy_async_smem();
  __syncthreads();

  // write-out: block 1 whole; block 2's rows that exist as partners: not row
  // n (slot 0 of pair 0, block-2 row np-1) and not row n/2 a second time (pair
  // n/2 of an even n, the last pair: block-2 row 0)
  const int j0 = (n_theta % 2 == 0 && p0 + np - 1 == n_theta / 2) ? 1 : 0;
  const int j1 = p0 == 0 ? np - 1 : np;
  if constexpr (G > 1) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();  // every copy of the band complete and visible cluster-wide
    uint32_t *copies[G];
#pragma unroll
    for (int c = 0; c < G; ++c) copies[c] = cl.map_shared_rank(slice_raw, c);
    unsigned long long best = 0ull;
    const uintptr_t fc0 = reinterpret_cast<uintptr_t>(frame) / SEG_BYTES;
    cluster_reduce_out<G, NWARPS>(p, dst1, mw1, ncell, copies, fc0, frame, rank, warp, lane,
                                  best);
    if (j1 > j0)
      cluster_reduce_out<G, NWARPS>(p, dst2 + j0 * n_rho, h2 + mw2 + j0 * n_rho,
                                    (j1 - j0) * n_rho, copies, fc0, frame, rank, warp, lane,
                                    best);
    if (p.hint_keys) {  // one key per CTA: the best cell it summed
      __shared__ unsigned long long s_best;
      if (tid == 0) s_best = 0ull;
      __syncthreads();
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other > best ? other : best;
      }
      if (lane == 0 && best) atomicMax(&s_best, best);
      __syncthreads();
      if (tid == 0) p.hint_keys[(static_cast<int64_t>(f) * p.n_bands + band) * G + rank] = s_best;
      if (f == 0 && band == 0 && tid == 0) write_hint_header(p, G);
    }
    cl.sync();  // no CTA leaves while another still reads its copy
    return;
  }
  bulk_rows_out(dst1, blk1, ncell, tid, NT);
  if (j1 > j0) bulk_rows_out(dst2 + j0 * n_rho, blk2 + j0 * n_rho, (j1 - j0) * n_rho, tid, NT);
  if (p.hint_keys) {
    SegBest best;
    const uintptr_t fc0 = reinterpret_cast<uintptr_t>(frame) / SEG_BYTES;
    uint32_t *segmax = p.segmax + static_cast<int64_t>(f) * p.n_seg;
    summarize_block(dst1, blk1, ncell, fc0, segmax, warp, NWARPS, lane, best);
    if (j1 > j0)
      summarize_block(dst2 + j0 * n_rho, blk2 + j0 * n_rho, (j1 - j0) * n_rho, fc0, segmax, warp,
                      NWARPS, lane, best);
    const unsigned long long key = seg_best_key(best, frame, lane);
    if (lane == 0) p.hint_keys[(static_cast<int64_t>(f) * p.n_bands + band) * NWARPS + warp] = key;
    if (f == 0 && band == 0 && tid == 0) write_hint_header(p, NWARPS);
  }
  if (tid == 0) bulk_wait_read();
}

int hough_plan_pairs(int n_theta, int n_rho, size_t smem_optin, int *ctas, int *ppb, int *n_bands,
                     size_t *smem_bytes) {
  const size_t fixed = sizeof(uint4) * HV_MAX_ROWS + 1024 + 64;
  const int np = hough_pair_count(n_theta);
  const size_t pair = static_cast<size_t>(n_rho) * 8u;
  auto plan = [&](size_t limit, int *nb) {
    int pmax = static_cast<int>(limit / pair);
    if (pmax > HV_MAX_ROWS) pmax = HV_MAX_ROWS;
    if (pmax < 1) return 0;
    *nb = (np + pmax - 1) / pmax;
    return (np + *nb - 1) / *nb;
  };
  int nb1 = 0, nb2 = 0;
  const int p1 = plan(smem_optin - fixed, &nb1);
  if (p1 < 1) return 0;
  const int p2 = plan(smem_optin / 2 - fixed, &nb2);
  const bool two = LD_HV_CTAS_MAX > 1 && p2 >= 4 && p1 >= 8;
  *ctas = two ? 2 : 1;
  *ppb = two ? p2 : p1;
  *n_bands = two ? nb2 : nb1;
  // two blocks of ppb rows, each shifted by up to 3 words and rounded to 16
  // bytes, + the scratch word (<= 52 bytes over 2 * ppb rows)
  *smem_bytes = ((static_cast<size_t>(*ppb) * pair + 15) / 16) * 16 + 64;
  return 1;
}

static AttrOnce g_pairs_attr[3];
static AttrOnce g_pairs_cl_attr[3][4];

// Thread-block clusters of G CTAs per band when one launch would otherwise
// occupy fewer than half the SMs (single frames): G = 8, 4 or 2, the largest
// that keeps the launch within one wave of the plan's CTA slots.
int hough_cluster_size(int batch, int n_bands, int ctas, int sm_count) {
  const int64_t ctas_total = static_cast<int64_t>(batch) * n_bands;
  const int64_t slots = static_cast<int64_t>(sm_count) * ctas;
  if (2 * ctas_total > static_cast<int64_t>(sm_count)) return 1;
  for (int g = 8; g >= 2; g >>= 1)
    if (ctas_total * g <= slots) return g;
  return 1;
}

template <int CTAS, int G>
static cudaError_t launch_pairs_cluster(const HoughParams &p, const TrigTable &trig,
                                        size_t smem_bytes, cudaStream_t stream, AttrOnce &attr) {
  auto kern = hough_vote_pairs_kernel<CTAS, G>;
  cudaError_t e = ensure_smem_attr(attr, kern, -(227 * 1024 / CTAS));
  if (e != cudaSuccess) return e;
  return launch_ex(kern, dim3(p.n_bands * G, p.batch), dim3(HV_THREADS / CTAS), smem_bytes, stream,
                   G, p, trig);
}

cudaError_t launch_hough_pairs(const HoughParams &p, const TrigTable &trig, int ctas,
                               size_t smem_bytes, cudaStream_t stream, int cluster) {
  if (cluster > 1) {
    const int gi = cluster == 8 ? 3 : cluster == 4 ? 2 : 1;
    AttrOnce &a = g_pairs_cl_attr[ctas][gi];
    cudaError_t e;
    if (ctas == 2)
      e = cluster == 8 ? launch_pairs_cluster<2, 8>(p, trig, smem_bytes, stream, a)
        : cluster == 4 ? launch_pairs_cluster<2, 4>(p, trig, smem_bytes, stream, a)
                       : launch_pairs_cluster<2, 2>(p, trig, smem_bytes, stream, a);
    else
      e = cluster == 8 ? launch_pairs_cluster<1, 8>(p, trig, smem_bytes, stream, a)
        : cluster == 4 ? launch_pairs_cluster<1, 4>(p, trig, smem_bytes, stream, a)
                       : launch_pairs_cluster<1, 2>(p, trig, smem_bytes, stream, a);
    if (e != cudaErrorLaunchOutOfResources && e != cudaErrorInvalidClusterSize) return e;
    // no room for the cluster (a partitioned or shared GPU): the per-band
    // kernel computes the same accumulator and hint
    cudaGetLastError();
  }
  auto kern = ctas == 2 ? hough_vote_pairs_kernel<2, 1> : hough_vote_pairs_kernel<1, 1>;
  cudaError_t e = ensure_smem_attr(g_pairs_attr[ctas], kern, -(227 * 1024 / ctas));
  if (e != cudaSuccess) return e;
  return launch_ex(kern, dim3(p.n_bands, p.batch), dim3(HV_THREADS / ctas), smem_bytes, stream, 1,
                   p, trig);
}

// ---------------------------------------------------------------------------
// B5: red.shared.add.u32 throughput.  1024 threads per CTA, 48 K-word array.
// The timed part is bracketed by clock64 in every CTA (cycles[] output), so
// the rate per clock per SM excludes the prologue and the checksum.
// ---------------------------------------------------------------------------
constexpr int AB_WORDS = 49152;

__global__ void __launch_bounds__(1024, 1)
    smem_atomic_bench_kernel(int mode, int iters, uint32_t *out) {
  extern __shared__ __align__(16) uint32_t buf[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < AB_WORDS; i += blockDim.x) buf[i] = 0u;
  __syncthreads();
  const long long c0 = clock64();
  const uint32_t base = smem_u32(buf);
  if (mode == 0) {
    // conflict-free, issue-free: lane l -> bank l, 32 distinct rows per
    // unrolled group addressed by immediate offsets, so the instruction
    // stream is (almost) pure ATOMS and the pipe itself is the limit
    const uint32_t a = base + ((static_cast<uint32_t>(warp) * 32u + lane) << 2);
    int i = 0;
    for (; i + 32 <= iters; i += 32) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        red_shared_add(a + j * 4096u, 1u);
    }
    for (; i < iters; ++i) red_shared_add(a, 1u);
  } else if (mode == 1) {
    uint32_t x = (blockIdx.x * 1024u + tid) * 2654435761u + 12345u;
#pragma unroll 8
    for (int i = 0; i < iters; ++i) {
      x = x * 1664525u + 1013904223u;
      red_shared_add(base + ((x >> 17) << 2), 1u);
    }
  } else {
#pragma unroll 8
    for (int i = 0; i < iters; ++i) red_shared_add(base + (static_cast<uint32_t>(warp) << 7), 1u);
  }
  __syncthreads();
  const long long c1 = clock64();
  if (tid < 32) {
    uint32_t s = 0;
    for (int i = tid; i < AB_WORDS; i += 32) s += buf[i];
    out[blockIdx.x * 34 + tid] = s;
  }
  if (tid == 0) {
    const unsigned long long dc = static_cast<unsigned long long>(c1 - c0);
    out[blockIdx.x * 34 + 32] = static_cast<uint32_t>(dc);
    out[blockIdx.x * 34 + 33] = static_cast<uint32_t>(dc >> 32);
  }
}

static AttrOnce g_bench_attr;

cudaError_t launch_smem_atomic_bench(int mode, int iters, int grid, uint32_t *scratch,
                                     cudaStream_t stream) {
  const int smem = AB_WORDS * 4;
  cudaError_t e = ensure_smem_attr(g_bench_attr, smem_atomic_bench_kernel, smem);
  if (e != cudaSuccess) return e;
  smem_atomic_bench_kernel<<<grid, 1024, smem, stream>>>(mode, iters, scratch);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ld
