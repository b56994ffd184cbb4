// ld_hough.cu -- B3: theta-partitioned shared-memory Hough voting, sm_100a;
//                B5: shared-memory atomic microbenchmark (the voting roofline).
//
// Paper: Eq. 3, voting, 180 one-degree PEs, the GPU
// design of one thread block per theta with the voting space in block shared
// memory and atomic adds for colliding votes.  DESIGN.md 6.2.
//
// Design: the paper gives each theta its own 48 KB block (K80).  On sm_100a a
// CTA owns a BAND of theta rows -- as many rows of n_rho uint32 counters as fit
// in the 227 KB opt-in shared memory -- so each frame's edge list is streamed
// n_theta / rows times instead of n_theta times.  Every thread holds 4 edges
// and, for each row of the band, issues one red.shared.add.u32 per edge at
// ((x*C + y*S + 2^14 + (D << 15)) >> 15) (SASS: ATOMS.POPC.INC).  The
// range proof done on the host (ld_api.cu) makes a per-vote bounds check
// unnecessary.  The band is then written to HBM with plain coalesced stores:
// no global atomics anywhere.
#include <cstdlib>

#include "ld_internal.cuh"

#ifndef LD_HV_UNROLL
#define LD_HV_UNROLL 4  // band rows per unrolled step
#endif

namespace ld {

// One block of 32 x EPL consecutive list entries of a warp (entry
// blk + 32j + lane in lane `lane`), voted into every row of the band.
template <int EPL, bool FULL>
// Entries past `end` (FULL = false) vote into the scratch word instead of
// being branched around: no divergent control flow in the tail.
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
    for (int j = 0; j < EPL; ++j)
    {
      const uint32_t a = ((xs[j] * k.x + ys[j] * k.y + k.z) >> 13) & ~3u;
      red_shared_add(FULL || ok[j] ? a : scratch, 1u);
    }
  }
}

template <int CTAS>
__global__ void __launch_bounds__(HV_THREADS / CTAS, CTAS)
    hough_vote_kernel(const HoughParams p, const __grid_constant__ TrigTable trig) {
  constexpr int NT = HV_THREADS / CTAS;
  extern __shared__ __align__(16) uint32_t slice_raw[];
  __shared__ uint4 rowk[HV_MAX_ROWS];  // per row: C, S, K = koff + (row address << 13)

  const int tid = threadIdx.x;
  const int band = blockIdx.x;
  const int f = blockIdx.y;
  const int t0 = band * p.rows_per_band;
  const int nr = min(p.rows_per_band, p.n_theta - t0);
  const int ncell = nr * p.n_rho;
  uint32_t *dst = p.acc + (static_cast<int64_t>(f) * p.n_theta + t0) * p.n_rho;
  // The slice starts at the same address modulo 16 as its destination, so the
  // write-out can be one bulk (TMA) copy of its 16-byte-aligned middle part.
  const int mw = static_cast<int>((reinterpret_cast<uintptr_t>(dst) & 15u) >> 2);
  uint32_t *slice = slice_raw + mw;
  const uint32_t sbase = smem_u32(slice);
  const uint32_t row_bytes = static_cast<uint32_t>(p.n_rho) * 4u;

  {
    uint4 *s4 = reinterpret_cast<uint4 *>(slice_raw);
    const int n4 = (mw + ncell + 3) >> 2;
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
  // the warps finish within one short block of each other.  At step j a
  // warp's 32 lanes hold the 32 consecutive entries blk + 32j + lane, which
  // the compaction made spatially compact (ld_sobel.cu): per theta they fall
  // into few consecutive rho bins, i.e. distinct banks, and equal bins merge
  // in ATOMS.POPC.INC.
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NWARPS = NT / 32;
  uint32_t base = 0;
  const uint32_t scratch = smem_u32(slice + ncell);  // inside the allocation, never written out
  for (; base + NWARPS * 32u * 16u <= n_edges; base += NWARPS * 32u * 16u)
    vote_block<16, true>(el, base + warp * 32u * 16u, n_edges, lane, nr, rowk, scratch);
  uint32_t blk = base + static_cast<uint32_t>(warp) * (32u * 8u);
  for (; blk + 32u * 8u <= n_edges; blk += NWARPS * 32u * 8u)
    vote_block<8, true>(el, blk, n_edges, lane, nr, rowk, scratch);
  if (blk < n_edges) vote_block<8, false>(el, blk, n_edges, lane, nr, rowk, scratch);
  __syncthreads();

  // write-out: unaligned head and tail words by threads, the aligned middle
  // by one bulk shared->global copy (async proxy: fence the ATOMS writes first)
  const int head = min((4 - mw) & 3, ncell);
  const int mid = ((ncell - head) >> 2) << 2;  // words, multiple of 4
  if (tid < head) dst[tid] = slice[tid];
  for (int i = head + mid + tid; i < ncell; i += NT) dst[i] = slice[i];
  if (tid == 0 && mid > 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + head),
                 "r"(smem_u32(slice + head)), "r"(static_cast<uint32_t>(mid) * 4u)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  if (p.hint_keys) {
    // Peak hint (DESIGN R25), while the bulk copy reads the slice: the band's
    // cells, row-major, split into one contiguous range per warp; for each
    // the largest count and its first cell.  Lanes scan with 16-byte loads
    // (the slice is 16-byte aligned at slice_raw); a lane keeps the first
    // vector where its running maximum rose, and the warp reduction keeps the
    // lowest cell index among equal counts.  No barrier: each warp writes its
    // own key.
    const int c0 = static_cast<int>((static_cast<int64_t>(ncell) * warp) / NWARPS);
    const int c1 = static_cast<int>((static_cast<int64_t>(ncell) * (warp + 1)) / NWARPS);
    const uint4 *v4 = reinterpret_cast<const uint4 *>(slice_raw);
    const int w0 = (mw + c0) >> 2, w1 = (mw + c1 + 3) >> 2;
    auto vec = [&](int w) {  // the vector's words outside [c0, c1) read as 0
      uint4 q = v4[w];
      const int i0 = w * 4 - mw;
      if (i0 < c0 || i0 + 4 > c1) {
        q.x = (i0 >= c0 && i0 < c1) ? q.x : 0u;
        q.y = (i0 + 1 >= c0 && i0 + 1 < c1) ? q.y : 0u;
        q.z = (i0 + 2 >= c0 && i0 + 2 < c1) ? q.z : 0u;
        q.w = (i0 + 3 >= c0 && i0 + 3 < c1) ? q.w : 0u;
      }
      return q;
    };
    uint32_t run = 0;
    int pos = -1;
    for (int w = w0 + lane; w < w1; w += 32) {
      const uint4 q = vec(w);
      const uint32_t m4 = max(max(q.x, q.y), max(q.z, q.w));
      if (m4 > run) {
        run = m4;
        pos = w;
      }
    }
    unsigned long long key = 0ull;
    if (run) {
      const uint4 q = vec(pos);
      const int j = q.x == run ? 0 : q.y == run ? 1 : q.z == run ? 2 : 3;
      const uint32_t idx = static_cast<uint32_t>(t0) * static_cast<uint32_t>(p.n_rho) +
                           static_cast<uint32_t>(pos * 4 + j - mw);
      key = (static_cast<unsigned long long>(run) << 32) | (0xFFFFFFFFu - idx);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
      key = other > key ? other : key;
    }
    if (lane == 0) p.hint_keys[(static_cast<int64_t>(f) * p.n_bands + band) * NWARPS + warp] = key;
    if (f == 0 && band == 0 && tid == 0) {
      uint32_t *h = p.hint_hdr;
      h[0] = HINT_MAGIC;
      h[1] = static_cast<uint32_t>(p.batch);
      h[2] = static_cast<uint32_t>(p.n_theta);
      h[3] = static_cast<uint32_t>(p.n_rho);
      h[4] = static_cast<uint32_t>(p.n_bands);
      h[5] = NWARPS;
    }
  }
  if (tid == 0 && mid > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
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
  // per CTA: the slice (+16 bytes of alignment shift), rowk, and a margin
  const size_t fixed = sizeof(uint4) * HV_MAX_ROWS + 1024 + 16;
  int nb1 = 0, nb2 = 0;
  const int r1 = rows_per_band(n_theta, n_rho, smem_optin - fixed, &nb1);
  if (r1 < 1) return 0;
  const int r2 = rows_per_band(n_theta, n_rho, smem_optin / 2 - fixed, &nb2);
  const bool two = r2 >= 8 && (smem_optin - fixed) / (static_cast<size_t>(n_rho) * 4u) >= 16;
  *ctas = two ? 2 : 1;
  *rpb = two ? r2 : r1;
  *n_bands = two ? nb2 : nb1;
  *smem_bytes = ((static_cast<size_t>(*rpb) * n_rho * 4 + 15) / 16) * 16 + 16;
  return 1;
}

static bool g_hough_attr[64][3];

cudaError_t launch_hough(const HoughParams &p, const TrigTable &trig, int ctas, size_t smem_bytes,
                         cudaStream_t stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = ctas == 2 ? hough_vote_kernel<2> : hough_vote_kernel<1>;
  if (!g_hough_attr[dev & 63][ctas]) {
    // the largest slice hough_plan can request for this CTA count, next to the
    // kernel's static shared memory (rowk, the hint reduction)
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024 / ctas - static_cast<int>(fa.sharedSizeBytes));
    if (e != cudaSuccess) return e;
    g_hough_attr[dev & 63][ctas] = true;
  }
  dim3 grid(p.n_bands, p.batch);
  kern<<<grid, HV_THREADS / ctas, smem_bytes, stream>>>(p, trig);
  note_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Half-angle paired voting (NEXT 2; the paper's Eq. 4-5): for a
// table with C[n-t] = -C[t] and S[n-t] = S[t], the rows t and n - t share
// Q = y*S[t] + K: V_t = Q + x*C[t], V_{n-t} = Q - x*C[t].  A CTA holds pairs
// p0 .. p0+np-1: rows t = p0 + i in the first half of its slice (in order,
// like the unpaired kernel), their partners n - t in the second half at the
// same slot i, i.e. a CONSTANT distance delta = rows_per_band * 4 n_rho bytes
// above, which the compiler folds into the ATOMS as a uniform-register offset
// ([R+UR]):
//   addr(t)   = ((x*C + Q) >> 13) & ~3          (Q = y*S + koff + (row t address << 13))
//   addr(n-t) = ((x*(-C) + Q) >> 13) & ~3, + delta
// 9 instructions per 2 votes instead of 10; consecutive bins stay in distinct
// banks.  Folding is exact as in the unpaired kernel: V in [0, 2^31) for both
// rows (host range proof, mirrored entries included), addresses < 2^18.
// Pair p = 0 and p = n/2 (n even) have no partner: their mirror votes land in
// a scratch row that is not written out.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int pair_partner(int t, int n_theta) {
  return (t == 0 || 2 * t == n_theta) ? -1 : n_theta - t;
}

int hough_pair_count(int n_theta) { return n_theta / 2 + 1; }

template <int EPL, bool FULL>
__device__ __forceinline__ void vote_block_pairs(const uint32_t *el, uint32_t blk, uint32_t end,
                                                 int lane, int np, const uint4 *rowk,
                                                 uint32_t delta, uint32_t scratch) {
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
#pragma unroll 2
  for (int r = 0; r < np; ++r) {
    const uint4 k = rowk[r];  // C, S, K, -C
#pragma unroll
    for (int j = 0; j < EPL; ++j)
    {
      const uint32_t q = ys[j] * k.y + k.z;
      const uint32_t a1 = ((xs[j] * k.x + q) >> 13) & ~3u;
      const uint32_t a2 = ((xs[j] * k.w + q) >> 13) & ~3u;
      red_shared_add(FULL || ok[j] ? a1 : scratch, 1u);
      red_shared_add((FULL || ok[j] ? a2 : scratch - delta) + delta, 1u);
    }
  }
}

template <int CTAS>
__global__ void __launch_bounds__(HV_THREADS / CTAS, CTAS)
    hough_vote_pairs_kernel(const HoughParams p, const __grid_constant__ TrigTable trig) {
  constexpr int NT = HV_THREADS / CTAS;
  constexpr int NWARPS = NT / 32;
  extern __shared__ __align__(16) uint32_t slice_raw[];
  __shared__ uint4 rowk[HV_MAX_ROWS];  // per pair: C, S, K = koff + (row t address << 13), -C

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int band = blockIdx.x;
  const int f = blockIdx.y;
  const int n_rho = p.n_rho, n_theta = p.n_theta;
  const int p0 = band * p.rows_per_band;
  const int np = min(p.rows_per_band, p.n_pairs - p0);
  const int ncell = np * n_rho;                       // first half (rows p0 ..)
  const int half = p.rows_per_band * n_rho;           // words to the partner half
  uint32_t *frame = p.acc + static_cast<int64_t>(f) * n_theta * n_rho;
  uint32_t *dst = frame + static_cast<int64_t>(p0) * n_rho;
  // first half at the destination's address modulo 16 (bulk write-out)
  const int mw = static_cast<int>((reinterpret_cast<uintptr_t>(dst) & 15u) >> 2);
  uint32_t *slice = slice_raw + mw;
  const uint32_t sbase = smem_u32(slice);
  const uint32_t row_bytes = static_cast<uint32_t>(n_rho) * 4u;
  const uint32_t delta = p.pair_delta;
  {
    uint4 *s4 = reinterpret_cast<uint4 *>(slice_raw);
    const int n4 = (mw + half + ncell + 3) >> 2;
    for (int i = tid; i < n4; i += NT) s4[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int i = tid; i < np; i += NT) {
      const int t = p0 + i;
      rowk[i] = make_uint4(static_cast<uint32_t>(trig.c[t]), static_cast<uint32_t>(trig.s[t]),
                           static_cast<uint32_t>(p.koff) + ((sbase + i * row_bytes) << 13),
                           static_cast<uint32_t>(-trig.c[t]));
    }
  }
  __syncthreads();

  const uint32_t n_edges = p.counts[f];
  const uint32_t *el = p.edges + static_cast<int64_t>(f) * p.edge_stride;
  // scratch word past the partner half (>= the partner offset): inside the
  // allocation, never written out
  const uint32_t scratch = smem_u32(slice + half + ncell);
  uint32_t base = 0;
  for (; base + NWARPS * 32u * 16u <= n_edges; base += NWARPS * 32u * 16u)
    vote_block_pairs<16, true>(el, base + warp * 32u * 16u, n_edges, lane, np, rowk, delta,
                               scratch);
  uint32_t blk = base + static_cast<uint32_t>(warp) * (32u * 8u);
  for (; blk + 32u * 8u <= n_edges; blk += NWARPS * 32u * 8u)
    vote_block_pairs<8, true>(el, blk, n_edges, lane, np, rowk, delta, scratch);
  if (blk < n_edges) vote_block_pairs<8, false>(el, blk, n_edges, lane, np, rowk, delta, scratch);
  __syncthreads();

  // write-out, first half: rows p0 .. p0+np-1 are consecutive in acc -- one
  // bulk copy of the aligned middle, head and tail words by threads
  const int head = min((4 - mw) & 3, ncell);
  const int mid = ((ncell - head) >> 2) << 2;
  if (tid < head) dst[tid] = slice[tid];
  for (int i = head + mid + tid; i < ncell; i += NT) dst[i] = slice[i];
  if (tid == 0 && mid > 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + head),
                 "r"(smem_u32(slice + head)), "r"(static_cast<uint32_t>(mid) * 4u)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  // second half: partner rows n - t descend as t ascends; coalesced thread
  // stores (the scratch partner of an unpaired row is dropped).  The peak
  // hint (R25) rides along here and scans the first half.
  const bool hint = p.hint_keys != nullptr;
  uint32_t run = 0, ridx = 0xFFFFFFFFu;
  for (int i = 0; i < np; ++i) {
    const int tp = pair_partner(p0 + i, n_theta);
    if (tp < 0) continue;  // uniform
    uint32_t *rb = frame + static_cast<int64_t>(tp) * n_rho;
    const uint32_t *src = slice + half + i * n_rho;
    const uint32_t ib = static_cast<uint32_t>(tp) * static_cast<uint32_t>(n_rho);
    for (int j = tid; j < n_rho; j += NT) {
      const uint32_t v = src[j];
      rb[j] = v;
      if (hint && v > run) {
        run = v;
        ridx = ib + static_cast<uint32_t>(j);
      }
    }
  }
  if (hint) {
    unsigned long long key = run ? (static_cast<unsigned long long>(run) << 32) | (0xFFFFFFFFu - ridx) : 0ull;
    // first half: this warp's contiguous share, 16-byte loads
    const int c0 = static_cast<int>((static_cast<int64_t>(ncell) * warp) / NWARPS);
    const int c1 = static_cast<int>((static_cast<int64_t>(ncell) * (warp + 1)) / NWARPS);
    const uint4 *v4 = reinterpret_cast<const uint4 *>(slice_raw);
    const int w0 = (mw + c0) >> 2, w1 = (mw + c1 + 3) >> 2;
    auto vec = [&](int w) {
      uint4 q = v4[w];
      const int i0 = w * 4 - mw;
      if (i0 < c0 || i0 + 4 > c1) {
        q.x = (i0 >= c0 && i0 < c1) ? q.x : 0u;
        q.y = (i0 + 1 >= c0 && i0 + 1 < c1) ? q.y : 0u;
        q.z = (i0 + 2 >= c0 && i0 + 2 < c1) ? q.z : 0u;
        q.w = (i0 + 3 >= c0 && i0 + 3 < c1) ? q.w : 0u;
      }
      return q;
    };
    uint32_t r2 = 0;
    int pos = -1;
    for (int w = w0 + lane; w < w1; w += 32) {
      const uint4 q = vec(w);
      const uint32_t m4 = max(max(q.x, q.y), max(q.z, q.w));
      if (m4 > r2) {
        r2 = m4;
        pos = w;
      }
    }
    if (r2) {
      const uint4 q = vec(pos);
      const int jj = q.x == r2 ? 0 : q.y == r2 ? 1 : q.z == r2 ? 2 : 3;
      const uint32_t idx = static_cast<uint32_t>(p0) * static_cast<uint32_t>(n_rho) +
                           static_cast<uint32_t>(pos * 4 + jj - mw);
      const unsigned long long k2 = (static_cast<unsigned long long>(r2) << 32) | (0xFFFFFFFFu - idx);
      key = k2 > key ? k2 : key;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
      key = other > key ? other : key;
    }
    if (lane == 0) p.hint_keys[(static_cast<int64_t>(f) * p.n_bands + band) * NWARPS + warp] = key;
    if (f == 0 && band == 0 && tid == 0) {
      uint32_t *h = p.hint_hdr;
      h[0] = HINT_MAGIC;
      h[1] = static_cast<uint32_t>(p.batch);
      h[2] = static_cast<uint32_t>(p.n_theta);
      h[3] = static_cast<uint32_t>(p.n_rho);
      h[4] = static_cast<uint32_t>(p.n_bands);
      h[5] = NWARPS;
    }
  }
  if (tid == 0 && mid > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

int hough_plan_pairs(int n_theta, int n_rho, size_t smem_optin, int *ctas, int *ppb, int *n_bands,
                     size_t *smem_bytes) {
  const size_t fixed = sizeof(uint4) * HV_MAX_ROWS + 1024 + 16;
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
  const char *env = getenv("LD_VOTE_CTAS");
  const bool two = env ? (env[0] == '2' && p2 >= 1) : (p2 >= 4 && p1 >= 8);
  *ctas = two ? 2 : 1;
  *ppb = two ? p2 : p1;
  *n_bands = two ? nb2 : nb1;
  *smem_bytes = ((static_cast<size_t>(*ppb) * pair + 15) / 16) * 16 + 16;
  return 1;
}

static bool g_pairs_attr[64][3];

cudaError_t launch_hough_pairs(const HoughParams &p, const TrigTable &trig, int ctas,
                               size_t smem_bytes, cudaStream_t stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = ctas == 2 ? hough_vote_pairs_kernel<2> : hough_vote_pairs_kernel<1>;
  if (!g_pairs_attr[dev & 63][ctas]) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024 / ctas - static_cast<int>(fa.sharedSizeBytes));
    if (e != cudaSuccess) return e;
    g_pairs_attr[dev & 63][ctas] = true;
  }
  dim3 grid(p.n_bands, p.batch);
  kern<<<grid, HV_THREADS / ctas, smem_bytes, stream>>>(p, trig);
  note_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// B5: red.shared.add.u32 throughput.  1024 threads per CTA, 48 K-word array.
// ---------------------------------------------------------------------------
constexpr int AB_WORDS = 49152;

__global__ void __launch_bounds__(1024, 1)
    smem_atomic_bench_kernel(int mode, int iters, uint32_t *out) {
  extern __shared__ __align__(16) uint32_t buf[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < AB_WORDS; i += blockDim.x) buf[i] = 0u;
  __syncthreads();
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
  if (tid < 32) {
    uint32_t s = 0;
    for (int i = tid; i < AB_WORDS; i += 32) s += buf[i];
    out[blockIdx.x * 32 + tid] = s;
  }
}

static bool g_bench_attr[64];

cudaError_t launch_smem_atomic_bench(int mode, int iters, int grid, uint32_t *scratch,
                                     cudaStream_t stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int smem = AB_WORDS * 4;
  if (!g_bench_attr[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(smem_atomic_bench_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    g_bench_attr[dev & 63] = true;
  }
  smem_atomic_bench_kernel<<<grid, 1024, smem, stream>>>(mode, iters, scratch);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ld
