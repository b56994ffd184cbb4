// ld_peaks.cu -- B4: deterministic Hough peaks (local max + top-K), sm_100a.
//
// Paper: "The line with the largest count value denotes the line with the most
// pixels on it. The process of picking the line with the most pixel value is
// called Hough Peak", done with MATLAB houghpeaks (Fig. 11).
// DESIGN R13/R14 make it deterministic: key(t, r) = (acc, -t, -r) encoded as
// the 64-bit integer (acc << 32) | (0xFFFFFFFF - (t*n_rho + r)); a cell is a
// candidate iff acc >= max(1, min_votes) and its key is the maximum of its
// (2ht+1) x (2hr+1) window clipped to the accumulator.  DESIGN.md 6.3.
//
// launch_peaks: first (windows of half_theta <= 12 and a window-cells x k
// product <= 2^20) peaks_fused_kernel, one CTA or cluster per frame: the
// certified bound from the peak hint (the voting kernel's, or one taken from
// acc by hint_from_acc_kernel), the sparse search over the chunks that can
// hold a top-k candidate, and the frame's top k (DESIGN R25, R30).  Frames it
// cannot settle -- and every frame with LD_PEAKS_DENSE -- go through a dense
// kernel, chosen per window (in this order):
//   peaks_warp_kernel    -- half_theta <= 3, 4 <= half_rho <= 64, k <= 64:
//                           every warp an independent strip x row chunk;
//   peaks_stream_kernel  -- half_theta <= 12: a CTA per strip x row chunk;
//   peaks_tile_kernel    -- separable window maximum over 16-row tiles
//                           (unrestricted searches);
//   peaks_band_kernel    -- generic fallback: a window scan per cell.
// All keep a per-unit top-k; peaks_merge_kernel (one CTA per frame) merges
// the per-unit lists.  The dense kernels skip the frames the fused search
// resolved; the warp and stream kernels start from its bound (gtau) and
// share a per-frame running threshold.
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "ld_internal.cuh"

// largest half_theta for which the streaming kernel loads 4 columns per thread
// (else 2); a build option (-DLD_PS_CPT4_MAX_HT=...) for experiments
#ifndef LD_PS_CPT4_MAX_HT
#define LD_PS_CPT4_MAX_HT 6
#endif

namespace ld {

typedef unsigned long long u64;

// Debug builds (LD_DEBUG=1 python -m paper_2212_09460_b200.build): indexed
// shared-memory writes of the streaming kernel are range-checked; a failed
// check records its source line (first one wins) and the write is skipped.
#ifdef LD_DEBUG
__device__ int g_ld_debug_line;
__device__ __forceinline__ bool ld_chk(bool ok, int line) {
  if (!ok) atomicCAS(&g_ld_debug_line, 0, line);
  return ok;
}
#define LD_CHK(c) ld_chk((c), __LINE__)
#else
#define LD_CHK(c) true
#endif

constexpr int PK_CHUNK = 2 * PK_THREADS;        // cells tested per round
constexpr int PK_BUF = PK_CHUNK + LD_MAX_K;     // candidate buffer (power of 2)
static_assert((PK_BUF & (PK_BUF - 1)) == 0, "PK_BUF must be a power of two");

__device__ __forceinline__ u64 mk_key(uint32_t v, uint32_t idx) {
  return (static_cast<u64>(v) << 32) | static_cast<u64>(0xFFFFFFFFu - idx);
}

// Per-frame threshold read: gpu-scope relaxed (a plain volatile load would be
// a system-scope strong load, a far longer round trip)
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// The sparse search (peaks_sparse_finish_kernel) already wrote this frame's
// peaks: the dense kernels skip it (uniform per CTA: f = blockIdx.y).
__device__ __forceinline__ bool frame_resolved(const PeaksParams &p, int f) {
  return p.resolved != nullptr && ld_relaxed_u32(p.resolved + f) != 0u;
}

// Sort a[0..n) descending (n a power of two); all threads participate.
__device__ void bitonic_desc(u64 *a, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const u64 x = a[i], y = a[ixj];
          const bool desc = (i & k) == 0;
          if (desc ? (x < y) : (x > y)) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

// buf[0..nbuf) holds new keys; merge top[0..*ntop) in and keep the best k.
// Must be called by all threads; ends synchronised.
__device__ void merge_topk(u64 *buf, int nbuf, u64 *top, int *ntop_s, int k) {
  const int ntop = *ntop_s;
  const int total = nbuf + ntop;
  int n = 1;
  while (n < total) n <<= 1;
  for (int i = threadIdx.x; i < ntop; i += blockDim.x) buf[nbuf + i] = top[i];
  for (int i = total + threadIdx.x; i < n; i += blockDim.x) buf[i] = 0ull;
  __syncthreads();
  bitonic_desc(buf, n);
  const int keep = total < k ? total : k;
  for (int i = threadIdx.x; i < keep; i += blockDim.x) top[i] = buf[i];
  __syncthreads();
  if (threadIdx.x == 0) *ntop_s = keep;
  __syncthreads();
}

__device__ __forceinline__ bool is_window_max(const uint32_t *A, int n_theta, int n_rho,
                                              int t, int r, uint32_t v, int ht, int hr) {
  const uint32_t idx = static_cast<uint32_t>(t * n_rho + r);
  const int ta = max(t - ht, 0), tb = min(t + ht, n_theta - 1);
  const int ra = max(r - hr, 0), rb = min(r + hr, n_rho - 1);
  for (int tt = ta; tt <= tb; ++tt) {
    const uint32_t *row = A + static_cast<int64_t>(tt) * n_rho;
    for (int rr = ra; rr <= rb; ++rr) {
      const uint32_t w = __ldg(row + rr);
      if (w > v) return false;
      if (w == v && static_cast<uint32_t>(tt * n_rho + rr) < idx) return false;
    }
  }
  return true;
}

__global__ void __launch_bounds__(PK_THREADS) peaks_band_kernel(const PeaksParams p) {
  LD_PDL_TRIGGER();
  pdl_wait();  // the previous kernel of the stream (acc, hint, flags) is complete
  __shared__ u64 buf[PK_BUF];
  __shared__ u64 top[LD_MAX_K];
  __shared__ int s_nbuf, s_ntop;

  const int band = blockIdx.x, f = blockIdx.y;
  if (frame_resolved(p, f)) return;
  const int t0 = p.cand_t0 + band * PK_ROWS;
  const int nr = min(PK_ROWS, p.cand_t1 - t0);
  const int ncell = nr * p.n_rho;
  const uint32_t *A = p.acc + static_cast<int64_t>(f) * p.n_theta * p.n_rho;

  if (threadIdx.x == 0) {
    s_nbuf = 0;
    s_ntop = 0;
  }
  __syncthreads();
  for (int base = 0; base < ncell; base += PK_CHUNK) {
    const u64 kth = (s_ntop == p.k) ? top[p.k - 1] : 0ull;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int c = base + threadIdx.x + j * PK_THREADS;
      if (c < ncell) {
        const int t = t0 + c / p.n_rho;
        const int r = c - (t - t0) * p.n_rho;
        const uint32_t v = __ldg(A + static_cast<int64_t>(t) * p.n_rho + r);
        if (v >= p.floor_votes) {
          const u64 key = mk_key(v, static_cast<uint32_t>((t + p.theta_offset) * p.n_rho + r));
          if (key > kth &&
              is_window_max(A, p.n_theta, p.n_rho, t, r, v, p.half_theta, p.half_rho)) {
            const int slot = atomicAdd(&s_nbuf, 1);
            buf[slot] = key;
          }
        }
      }
    }
    __syncthreads();
    const int nbuf = s_nbuf;
    if (nbuf > 0) {
      merge_topk(buf, nbuf, top, &s_ntop, p.k);
      if (threadIdx.x == 0) s_nbuf = 0;
    }
    __syncthreads();
  }
  u64 *out = p.band_keys + (static_cast<int64_t>(f) * p.n_units + band) * p.k;
  const int ntop = s_ntop;
  for (int i = threadIdx.x; i < p.k; i += PK_THREADS) out[i] = i < ntop ? top[i] : 0ull;
}

// ---------------------------------------------------------------------------
// Fused hinted search (DESIGN R25 + R30, one CTA per frame, one launch): the
// bound, the sparse search and its top k without a global round trip or a
// launch between them -- what bounds a single frame's latency.
//   1. bound: the voting kernel's range maxima are sorted (bitonic: shuffles
//      for partners inside a warp, shared memory across warps) and verified
//      32 at a time, one warp per key, against the full candidate definition;
//      the value of the k-th verified key in key order bounds the frame's
//      k-th best candidate from below (tau_f; 0 if fewer than k verify or a
//      key below the floor ends the list first);
//   2. sparse: every cell >= tau_f lies in a 1 KB chunk whose recorded maximum
//      is >= tau_f; the verified keys >= tau_f are candidates already; the
//      chunks are read one per warp and their other cells >= tau_f checked
//      lane-parallel against their (up to 8) neighbours inside the window (a
//      necessary condition); the survivors, pooled, are dealt to the warps for
//      the exact test (the +-1-row, +-15-column neighbourhood first, where
//      most of them fail, then the whole window);
//   3. the candidates (all >= tau_f, at least the k verified ones) are sorted
//      and the best k written: peaks, n_peaks, resolved = 1.
// A frame it cannot finish (no or mismatched hint, chunk maxima of another
// accumulator, fewer than k verified, queue or list overflow) keeps
// resolved = 0 and gets gtau = tau_f (possibly 0): the dense kernels launched
// after it start from that bound.  Without p.resolved (dense-only searches)
// only the bound is computed.
// ---------------------------------------------------------------------------
// -DLD_PF_STATS=1 (experiments): per-frame phase clocks and counts into the
// workspace's diagnostics area (diag[f][0..11], tools/pf_stats.py)
#ifndef LD_PF_STATS
#define LD_PF_STATS 0
#endif
constexpr int PF_KEYS = 2048;   // range maxima sorted per frame (more are combined)
constexpr int PF_QUEUE = 4096;  // hot chunks per pass
constexpr int PF_SURV = 2048;   // prefilter survivors per pass
static_assert(SP_CAP == 2048, "candidate list size");
// dynamic shared memory: keys, candidates, survivors (u64) + queue (int)
constexpr size_t PF_SMEM = sizeof(u64) * (PF_KEYS + SP_CAP + PF_SURV) + sizeof(int) * PF_QUEUE;

// Exact window test of cell idx = (t, r), value v, by one warp: A[idx] == v,
// every count of the clipped window is <= v and an equal one sits at a higher
// index -- i.e. the cells before idx in (theta, rho) order are < v and the
// cells after it <= v.  NEAR: the +-1-row, +-15-column neighbourhood first
// (one load per lane and row), where most non-maxima fail.  Then the centre
// row cell by cell, then the other rows as 16-byte vectors (each row's cells
// [ra, rb] from the aligned vector holding ra on; U vectors in flight per
// lane, (row, vector) advancing incrementally): one maximum per vector, into
// the maximum above or below the centre row.  A vector reaching outside the
// frame's cells (misaligned frame edges) is read cell by cell.  Cell indices
// within a frame fit 32 bits (n_theta * n_rho < 2^31, checked by the host).
// part / parts: a team of `parts` warps shares one test -- warp `part` takes
// the non-centre rows q with q % parts == part (and part 0 the NEAR check and
// the centre row); the cell is a window maximum iff every part returns true.
template <int U, bool NEAR>
__device__ __forceinline__ bool warp_window_max(const uint32_t *A, int64_t ncells, int n_theta,
                                                int n_rho, int t, int r, uint32_t v, int ht,
                                                int hr, int lane, int part = 0, int parts = 1) {
  const int idx = t * n_rho + r;
  const int ta = max(t - ht, 0), tb = min(t + ht, n_theta - 1);
  const int ra = max(r - hr, 0), rb = min(r + hr, n_rho - 1);
  const int nc = static_cast<int>(ncells);
  if (NEAR && part == 0) {
    const int dr = lane - 15;  // lanes 0..30: columns r-15 .. r+15
    const bool col = lane < 31 && r + dr >= ra && r + dr <= rb;
    uint32_t w[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int tt = t - 1 + d;
      w[d] = (col && tt >= ta && tt <= tb) ? __ldg(A + (idx + (d - 1) * n_rho + dr)) : 0u;
    }
    bool bad = false;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      bad |= w[d] > v || (w[d] == v && (d < 1 || (d == 1 && dr < 0))) ||
             (d == 1 && dr == 0 && w[d] != v);
    if (__any_sync(0xffffffffu, bad)) return false;
  }
  if (part == 0) {  // the centre row: before r < v, after r <= v, at r == v
    bool bad = false;
    const int row0 = t * n_rho;
#pragma unroll 4
    for (int c = ra + lane; c <= rb; c += 32) {
      const uint32_t w = __ldg(A + row0 + c);
      bad |= c < r ? w >= v : (c > r ? w > v : w != v);  // no short circuit: loads overlap
    }
    if (__any_sync(0xffffffffu, bad)) return false;
  }
  // rows other than the centre one, this part's share: q = part + parts * i
  const int rows = part < tb - ta ? (tb - ta - part + parts - 1) / parts : 0;
  if (rows == 0) return true;
  const int nv = (rb - ra + 3) / 4 + 1;  // vectors per row, at any alignment
  const int items = rows * nv;
  const int sh = static_cast<int>((reinterpret_cast<uintptr_t>(A) >> 2) & 3u);  // A's word offset mod 4
  auto row_of = [&](int qi) {  // the part's qi-th row
    const int qq = part + parts * qi;
    return ta + qq + (ta + qq >= t ? 1 : 0);
  };
  // first cell of the aligned vector holding cell ra of row tt (frame index)
  auto first_vec = [&](int tt) {
    const int c = tt * n_rho + ra;
    return c - ((c + sh) & 3);
  };
  // item 32 u + lane of each step, as (q-th non-centre row, vector j): U
  // independent chains advancing by 32 U items per step
  const int dq = 32 * U / nv, dj = 32 * U - dq * nv;
  int qs[U], js[U], tts[U], a0s[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    qs[u] = (32 * u + lane) / nv;
    js[u] = 32 * u + lane - qs[u] * nv;
    tts[u] = row_of(qs[u]);
    a0s[u] = first_vec(tts[u]);
  }
  uint32_t above = 0u, below = 0u;  // maxima over the rows above / below t
  const int safe = (4 - sh) & 3;  // the frame's first 16-byte-aligned cell
  for (int i0 = 0; i0 < items; i0 += 32 * U) {
    uint4 w[U];
    int lo[U], hi[U], c4[U];  // in-window cells of vector u: e in [lo, hi]
    bool up[U];
    bool edge = false;  // a vector reaching outside the frame's cells
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c4[u] = a0s[u] + 4 * js[u];
      const int col0 = c4[u] - tts[u] * n_rho;
      const bool live = i0 + 32 * u + lane < items && col0 <= rb;
      lo[u] = ra - col0;
      hi[u] = live ? rb - col0 : -1;
      up[u] = tts[u] < t;
      edge |= live && (c4[u] < 0 || c4[u] + 4 > nc);
      if (!live) c4[u] = safe;
      qs[u] += dq;
      js[u] += dj;
      if (js[u] >= nv) {
        js[u] -= nv;
        ++qs[u];
      }
      tts[u] = row_of(qs[u]);
      a0s[u] = first_vec(tts[u]);
    }
    if (!__any_sync(0xffffffffu, edge)) {  // all U vectors of every lane in flight at once
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] = __ldg(reinterpret_cast<const uint4 *>(A + c4[u]));
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c4[u];
        w[u].x = c + 0 >= 0 && c + 0 < nc ? __ldg(A + c + 0) : 0u;
        w[u].y = c + 1 >= 0 && c + 1 < nc ? __ldg(A + c + 1) : 0u;
        w[u].z = c + 2 >= 0 && c + 2 < nc ? __ldg(A + c + 2) : 0u;
        w[u].w = c + 3 >= 0 && c + 3 < nc ? __ldg(A + c + 3) : 0u;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t m01 = max(0 >= lo[u] && 0 <= hi[u] ? w[u].x : 0u,
                               1 >= lo[u] && 1 <= hi[u] ? w[u].y : 0u);
      const uint32_t m23 = max(2 >= lo[u] && 2 <= hi[u] ? w[u].z : 0u,
                               3 >= lo[u] && 3 <= hi[u] ? w[u].w : 0u);
      const uint32_t mv = max(m01, m23);
      above = max(above, up[u] ? mv : 0u);
      below = max(below, up[u] ? 0u : mv);
    }
    if (__any_sync(0xffffffffu, above >= v || below > v)) return false;
  }
  return true;
}

// Necessary condition for cell idx = (t, r) with value v: it beats its
// neighbours at distance 1 that lie inside its window (dt within ht, dr within
// hr) and inside the accumulator -- by value, or by index on a tie.  One
// lane, all loads independent.
__device__ __forceinline__ bool beats_neighbours(const uint32_t *A, int n_theta, int n_rho, int t,
                                                 int r, uint32_t v, int ht, int hr) {
  const int64_t idx = static_cast<int64_t>(t) * n_rho + r;
  uint32_t w[8];
  bool in[8];
  int j = 0;
#pragma unroll
  for (int dt = -1; dt <= 1; ++dt) {
#pragma unroll
    for (int dr = -1; dr <= 1; ++dr) {
      if (dt == 0 && dr == 0) continue;
      in[j] = (dt == 0 || ht > 0) && (dr == 0 || hr > 0) && t + dt >= 0 && t + dt < n_theta &&
              r + dr >= 0 && r + dr < n_rho;
      w[j] = in[j] ? __ldg(A + idx + dt * n_rho + dr) : 0u;
      ++j;
    }
  }
  bool ok = true;
  j = 0;
#pragma unroll
  for (int dt = -1; dt <= 1; ++dt) {
#pragma unroll
    for (int dr = -1; dr <= 1; ++dr) {
      if (dt == 0 && dr == 0) continue;
      const bool lower = dt < 0 || (dt == 0 && dr < 0);  // neighbour index below idx
      ok = ok && !(in[j] && (w[j] > v || (w[j] == v && lower)));
      ++j;
    }
  }
  return ok;
}

// Sort a[0..n2) descending, n2 a power of two in [32, NT * S]: element e lives
// in register x[e / NT] of thread e % NT; compare-exchange partners inside a
// warp go through shuffles (run only by the warps that hold elements, all
// consecutive stages j < 32 of one k in a row), across warps through shared
// memory (a), across register slots in place.  Returns with a[] holding the
// sorted keys.
template <int NT, int S>
__device__ __forceinline__ void block_sort_desc(u64 *a, int n2, u64 (&x)[S]) {
  static_assert(S <= 4, "at most 4 slots");
  const int tid = threadIdx.x, wbase = tid & ~31;
  auto cx = [&](u64 &lo_slot, u64 &hi_slot, int s, int k) {  // in-thread pair
    const int e = s * NT + tid;
    if (e < n2) {
      const bool desc = (e & k) == 0;
      const u64 hi = lo_slot > hi_slot ? lo_slot : hi_slot, lo = lo_slot > hi_slot ? hi_slot : lo_slot;
      lo_slot = desc ? hi : lo;
      hi_slot = desc ? lo : hi;
    }
  };
  for (int k = 2; k <= n2; k <<= 1) {
    int j = k >> 1;
    for (; j >= NT; j >>= 1) {  // partner in another slot of this thread
      if (j == NT) {
        if (S > 1) cx(x[0], x[1 % S], 0, k);
        if (S > 3) cx(x[2 % S], x[3 % S], 2, k);
      } else if (S > 3) {
        cx(x[0], x[2 % S], 0, k);
        cx(x[1 % S], x[3 % S], 1, k);
      }
    }
    for (; j >= 32; j >>= 1) {  // partner in another warp
#pragma unroll
      for (int s = 0; s < S; ++s)
        if (s * NT + tid < n2) a[s * NT + tid] = x[s];
      __syncthreads();
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int e = s * NT + tid;
        if (e < n2) {
          const u64 o = a[e ^ j];
          const bool desc = (e & k) == 0, lower = (e & j) == 0;
          const u64 hi = x[s] > o ? x[s] : o, lo = x[s] > o ? o : x[s];
          x[s] = (desc == lower) ? hi : lo;
        }
      }
      __syncthreads();
    }
    if (wbase < n2) {  // partners in this warp: stages j .. 1
#pragma unroll
      for (int jj = 16; jj > 0; jj >>= 1) {
        if (jj <= j) {
#pragma unroll
          for (int s = 0; s < S; ++s) {
            if (s * NT + wbase < n2) {  // warp-uniform
              const int e = s * NT + tid;
              const u64 o = __shfl_xor_sync(0xffffffffu, x[s], jj);
              const bool desc = (e & k) == 0, lower = (e & jj) == 0;
              const u64 hi = x[s] > o ? x[s] : o, lo = x[s] > o ? o : x[s];
              x[s] = (desc == lower) ? hi : lo;
            }
          }
        }
      }
    }
  }
#pragma unroll
  for (int s = 0; s < S; ++s)
    if (s * NT + tid < n2) a[s * NT + tid] = x[s];
  __syncthreads();
}

// Bitonic networks over L = 32 * M keys held by one warp, element e = 32 i +
// lane in y[i]: partners inside the warp through shuffles, across registers
// in place (all indices static).
template <int M>
__device__ __forceinline__ void cx_lane(u64 &y, int e, int j, bool desc, int lane) {
  const u64 o = __shfl_xor_sync(0xffffffffu, y, j);
  const bool lower = (e & j) == 0;
  const u64 hi = y > o ? y : o, lo = y > o ? o : y;
  y = (desc == lower) ? hi : lo;
}
template <int M>
__device__ __forceinline__ void cx_regs(u64 &a, u64 &b, bool desc) {  // a holds the lower element
  const u64 hi = a > b ? a : b, lo = a > b ? b : a;
  a = desc ? hi : lo;
  b = desc ? lo : hi;
}
// sort descending
template <int M>
__device__ __forceinline__ void warp_sort_desc(u64 (&y)[M], int lane) {
#pragma unroll
  for (int k = 2; k <= 32 * M; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
#pragma unroll
        for (int i = 0; i < M; ++i)
          if ((i & (j >> 5)) == 0) cx_regs<M>(y[i], y[i | (j >> 5)], ((32 * i + lane) & k) == 0);
      } else {
#pragma unroll
        for (int i = 0; i < M; ++i) cx_lane<M>(y[i], 32 * i + lane, j, ((32 * i + lane) & k) == 0, lane);
      }
    }
  }
}
// a bitonic sequence into descending order
template <int M>
__device__ __forceinline__ void warp_merge_desc(u64 (&y)[M], int lane) {
#pragma unroll
  for (int j = 16 * M; j > 0; j >>= 1) {
    if (j >= 32) {
#pragma unroll
      for (int i = 0; i < M; ++i)
        if ((i & (j >> 5)) == 0) cx_regs<M>(y[i], y[i | (j >> 5)], true);
    } else {
#pragma unroll
      for (int i = 0; i < M; ++i) cx_lane<M>(y[i], 32 * i + lane, j, true, lane);
    }
  }
}

// The best L = 32 * M keys of a[0..n2) (n2 a power of two >= L), sorted
// descending into a[0..L): every warp sorts L-key chunks in registers, then a
// tree merges chunk pairs keeping the better half -- the elementwise maximum
// of one sorted list and the other reversed is a bitonic sequence holding
// the best L of both, which one bitonic merge sorts.  All threads call; ends
// synchronised.  (A full sort of the 184 .. 2048 range maxima costs 4-19x
// more: cross-warp stages at every level.)
template <int NT, int M>
__device__ void block_top_desc(u64 *a, int n2) {
  constexpr int NW = NT / 32, L = 32 * M;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int C = n2 / L;
  for (int c = warp; c < C; c += NW) {
    u64 y[M];
#pragma unroll
    for (int i = 0; i < M; ++i) y[i] = a[c * L + 32 * i + lane];
    warp_sort_desc<M>(y, lane);
#pragma unroll
    for (int i = 0; i < M; ++i) a[c * L + 32 * i + lane] = y[i];
  }
  __syncthreads();
  for (int st = 1; st < C; st <<= 1) {
    for (int c = warp * 2 * st; c < C; c += NW * 2 * st) {
      u64 y[M];
#pragma unroll
      for (int i = 0; i < M; ++i) {
        const u64 u = a[c * L + 32 * i + lane], z = a[(c + st) * L + (L - 1 - (32 * i + lane))];
        y[i] = u > z ? u : z;
      }
      warp_merge_desc<M>(y, lane);
#pragma unroll
      for (int i = 0; i < M; ++i) a[c * L + 32 * i + lane] = y[i];
    }
    __syncthreads();
  }
}

// position of key in a[0..n) sorted descending (distinct keys), or -1
__device__ __forceinline__ int find_desc(const u64 *a, int n, u64 key) {
  int lo = 0, hi = n;  // a[lo-1] > key >= a[hi]... invariant: answer in [lo, hi)
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] > key) lo = mid + 1;
    else hi = mid;
  }
  return lo < n && a[lo] == key ? lo : -1;
}

// Cluster plumbing of the fused search: G CTAs of one frame (a thread-block
// cluster) split the verification keys and the chunk maxima; CTA 0 of the
// cluster gathers the candidates (distributed shared memory) and writes the
// frame's peaks.  G = 1 is the plain one-CTA-per-frame kernel.
template <int G>
__device__ __forceinline__ void pf_sync() {
  if constexpr (G > 1) cooperative_groups::this_cluster().sync();
  else __syncthreads();
}
template <int G, typename T>
__device__ __forceinline__ T *pf_at(T *p, int rank) {  // p in CTA `rank` of the cluster
  if constexpr (G > 1) return cooperative_groups::this_cluster().map_shared_rank(p, rank);
  else return p;
}

template <int NT, int G, int MINB>
__global__ void __launch_bounds__(NT, MINB) peaks_fused_kernel(const PeaksParams p) {
  LD_PDL_TRIGGER();
  pdl_wait();  // the previous kernel of the stream (acc, hint, flags) is complete
  constexpr int NW = NT / 32;
  constexpr int S = PF_KEYS / NT;
  // window-test vectors in flight per lane (the register budget; 8 measured no faster)
  constexpr int WU = MINB > 1 ? 2 : 4;
  static_assert(NW <= 32, "warp 0 reads one result per lane of each 32-key chunk");
  extern __shared__ __align__(16) unsigned char pf_smem[];
  u64 *keys = reinterpret_cast<u64 *>(pf_smem);  // sorted range maxima
  u64 *cand = keys + PF_KEYS;                     // candidate keys (CTA 0)
  u64 *surv = cand + SP_CAP;                      // prefilter survivors
  int *queue = reinterpret_cast<int *>(surv + PF_SURV);
  __shared__ uint32_t s_vbits[PF_KEYS / 32];      // verified keys (by sorted position)
  __shared__ int s_ok[2][NW];                     // a round's results, by parity
  __shared__ int s_pok[NW];                       // the parts of the survivors' tests
  __shared__ int s_state, s_found, s_nq, s_ncand, s_nsurv, s_last, s_fail;
  __shared__ uint32_t s_tau;
  const int rank = G > 1 ? static_cast<int>(blockIdx.x % G) : 0;
  const int f = blockIdx.x / G, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_theta = p.n_theta, n_rho = p.n_rho;
  const uint32_t *h = p.hint_hdr;
  const bool match = h[0] == HINT_MAGIC && h[1] == static_cast<uint32_t>(p.batch) &&
                     h[2] == static_cast<uint32_t>(n_theta) &&
                     h[3] == static_cast<uint32_t>(n_rho) && h[5] >= 1 &&
                     h[5] <= HINT_MAX_RANGES && h[4] >= 1 && h[4] <= static_cast<uint32_t>(n_theta) &&
                     h[6] == static_cast<uint32_t>(p.n_seg);
  // the chunk maxima describe the accumulator at the address voting wrote it
  // to: a copy elsewhere keeps the (verified) bound but not the sparse search
  const uint64_t acc_addr = reinterpret_cast<uintptr_t>(p.acc);
  const bool sparse = match && p.resolved != nullptr && p.segmax != nullptr &&
                      h[7] == static_cast<uint32_t>(acc_addr) &&
                      h[8] == static_cast<uint32_t>(acc_addr >> 32);
  const int n_src = match ? static_cast<int>(h[4] * h[5]) : 0;
  const int64_t ncells = static_cast<int64_t>(n_theta) * n_rho;
  const uint32_t *A = p.acc + static_cast<int64_t>(f) * ncells;
  const int ht = p.half_theta, hr = p.half_rho;
#if LD_PF_STATS
  long long st_t0 = clock64(), st_t1 = 0, st_t2 = 0, st_t3 = 0, st_tl = 0;
  __shared__ int st_hot, st_surv, st_rounds;
  __shared__ long long st_lat, st_win;
  if (tid == 0) {
    st_hot = st_surv = st_rounds = 0;
    st_lat = st_win = 0;
  }
#endif

  // ---- 1. the bound
  // the keys are verified in key order from the best L = 32 m (m from k: the
  // k-th verified key sat within the best 2k on the road workloads); past
  // them, all n are sorted and the rounds go on
  const int m = p.k <= 16 ? 1 : p.k <= 32 ? 2 : 4;
  // more keys than the selection takes (2048; 512 for k <= 16, where the
  // best 32 decide): combine g consecutive ranges (the maximum of a union of
  // ranges is a cell of the accumulator all the same)
  const int cap = m == 1 ? 512 : PF_KEYS;
  const int g = (n_src + cap - 1) / cap;
  const int n = n_src > 0 ? (n_src + g - 1) / g : 0;
  int n2 = 32 * m;
  while (n2 < n) n2 <<= 1;
  const u64 *src = p.hint_keys + static_cast<int64_t>(f) * n_src;
  auto load_keys = [&](u64 (&x)[S]) {
    if (g == 1) {  // every slot's load in flight at once
#pragma unroll
      for (int s = 0; s < S; ++s) x[s] = s * NT + tid < n ? __ldg(src + s * NT + tid) : 0ull;
    } else {
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int i = s * NT + tid;
        u64 mx = 0ull;
        if (i < n)
          for (int j = i * g; j < min(i * g + g, n_src); ++j) mx = src[j] > mx ? src[j] : mx;
        x[s] = mx;
      }
    }
  };
  {
    u64 x[S];
    load_keys(x);
#if LD_PF_STATS
    st_tl = clock64();
#endif
#pragma unroll
    for (int s = 0; s < S; ++s)
      if (s * NT + tid < n2) keys[s * NT + tid] = x[s];
    if (tid < PF_KEYS / 32) s_vbits[tid] = 0u;
    if (tid == 0) {
      s_state = n > 0 ? 0 : 2;
      s_found = 0;
      s_tau = 0u;
      s_nq = 0;
      s_ncand = 0;
      s_nsurv = 0;
      s_last = 0;
      s_fail = 0;
    }
    __syncthreads();
    if (m == 1) block_top_desc<NT, 1>(keys, n2);
    else if (m == 2) block_top_desc<NT, 2>(keys, n2);
    else block_top_desc<NT, 4>(keys, n2);
  }
#if LD_PF_STATS
  st_t1 = clock64();
#endif
  // rounds of RW keys in key order (all the cluster's warps, at most the best
  // L per round, at most 128); key r0 + i is tested by warp i / G of the
  // cluster's CTA i % G, the results read cluster-wide
  int limit = 32 * m;  // keys[0..limit) are in key order
  const int RW = min(min(NW * G, 128), limit);
  int par = 0;
  for (int r0 = 0; s_state == 0; r0 += RW, par ^= 1) {
#if LD_PF_STATS
    if (tid == 0) ++st_rounds;
#endif
    if (r0 >= limit) {  // past the best L: sort them all (the first L stay in place)
      u64 x[S];
      load_keys(x);
      block_sort_desc<NT, S>(keys, n2, x);
      limit = n2;
    }
    const int i = warp * G + rank;
    if (i < RW) {
      const int j = r0 + i;
      const u64 key = j < n2 ? keys[j] : 0ull;
      const uint32_t v = static_cast<uint32_t>(key >> 32);
      int ok = -1;  // below the floor or exhausted: this and every later key end the search
      if (key != 0ull && v >= p.floor_votes) {
        const uint32_t idx = 0xFFFFFFFFu - static_cast<uint32_t>(key);
        const int t = static_cast<int>(idx / static_cast<uint32_t>(n_rho));
        const int r = static_cast<int>(idx - static_cast<uint32_t>(t) * n_rho);
#if LD_PF_STATS
        long long l0 = clock64();
        const uint32_t probe = __ldg(A + idx);
        long long l1 = clock64() + (probe == 0xFFFFFFFFu ? 1 : 0);
#endif
        // (a cell outside the candidate rows is no candidate of this search)
        ok = (t >= p.cand_t0 && t < p.cand_t1 &&
              warp_window_max<WU, false>(A, ncells, n_theta, n_rho, t, r, v, ht, hr, lane)) ? 1 : 0;
#if LD_PF_STATS
        long long l2 = clock64();
        if (warp == 0 && lane == 0 && r0 == 0) {
          st_lat = l1 - l0;
          st_win = l2 - l1;
        }
#endif
      }
      if (lane == 0) s_ok[par][warp] = ok;
    }
    pf_sync<G>();
    if (warp == 0) {
      // the round's results 32 keys at a time, in key order, up to the decision
      for (int c0 = 0; c0 < RW; c0 += 32) {
        const int ii = c0 + lane;  // key r0 + ii: warp ii / G of CTA ii % G
        const int o = ii < RW ? *pf_at<G>(&s_ok[par][ii / G], ii % G) : 0;
        const uint32_t endm = __ballot_sync(0xffffffffu, o < 0);
        uint32_t okm = __ballot_sync(0xffffffffu, o > 0);
        if (endm) okm &= (1u << (__ffs(endm) - 1)) - 1u;  // verified keys before the end
        const int need = p.k - s_found;
        const int c = __popc(okm);
        bool done = false;
        if (c >= need) {  // the need-th verified key sets the bound
          const bool me = ((okm >> lane) & 1u) && __popc(okm & ((2u << lane) - 1u)) == need;
          const uint32_t who = __ballot_sync(0xffffffffu, me);
          okm &= (2u << (__ffs(who) - 1)) - 1u;  // up to and including it
          if (lane == 0) {
            s_tau = static_cast<uint32_t>(keys[r0 + c0 + __ffs(who) - 1] >> 32);
            s_state = 1;
          }
          done = true;
        } else {
          if (lane == 0) s_found += c;
          done = endm != 0u;  // (keys past the list read as 0: an end)
          if (done && lane == 0) s_state = 2;
        }
        // verified positions (rounds start at multiples of min(RW, 32))
        if (lane == 0) s_vbits[(r0 + c0) >> 5] |= okm << ((r0 + c0) & 31);
        __syncwarp();
        if (done) break;
      }
      if (lane == 0) {
        s_last = r0 + RW;
        if (s_state == 0 && r0 + RW >= n2) s_state = 2;
      }
    }
    __syncthreads();
  }
  // every CTA has read every CTA's last round (its s_ok stays live until here)
  if (G > 1) pf_sync<G>();
  const uint32_t tau_f = s_tau;  // 0 = no bound; the same in every CTA of the cluster
#if LD_PF_STATS
  st_t2 = clock64();
#endif
  if (tau_f == 0u || !sparse) {
    if (tid == 0 && rank == 0) {
      p.gtau[f] = tau_f;
      if (p.resolved) p.resolved[f] = 0u;
    }
    return;
  }

  // ---- 2. the sparse search over the chunks whose maximum reaches tau (the
  // chunk maxima split over the cluster's CTAs; candidates gathered in CTA 0)
  const uint32_t tau = tau_f > p.floor_votes ? tau_f : p.floor_votes;
  const int nv = min(s_last, n2);
  int *ncand0 = pf_at<G>(&s_ncand, 0);
  u64 *cand0 = pf_at<G>(cand, 0);
  int *fail0 = pf_at<G>(&s_fail, 0);
  // the verified keys (all >= tau: verified in key order up to the k-th) are
  // candidates; the chunk scan skips them
  if (rank == 0)
    for (int i = tid; i < nv; i += NT)
      if ((s_vbits[i >> 5] >> (i & 31)) & 1u) cand[atomicAdd(&s_ncand, 1)] = keys[i];
  const uint32_t *Sg = p.segmax + static_cast<int64_t>(f) * p.n_seg;
  const uintptr_t c0 = reinterpret_cast<uintptr_t>(A) / SEG_BYTES;
  // the chunks of the candidate rows [cand_t0, cand_t1), split over the cluster
  const int64_t rc0 = static_cast<int64_t>(p.cand_t0) * n_rho, rc1 = static_cast<int64_t>(p.cand_t1) * n_rho;
  const uintptr_t a_addr = reinterpret_cast<uintptr_t>(A);
  const int qa = static_cast<int>((a_addr + 4 * rc0) / SEG_BYTES - c0);
  const int qb = rc1 > rc0 ? static_cast<int>((a_addr + 4 * (rc1 - 1)) / SEG_BYTES - c0) + 1 : qa;
  const int q_lo = qa + static_cast<int>(static_cast<int64_t>(qb - qa) * rank / G);
  const int q_hi = qa + static_cast<int>(static_cast<int64_t>(qb - qa) * (rank + 1) / G);
  bool fail = false;  // CTA-uniform
  constexpr int SCAN = 8 * NT;  // chunk maxima per batch, 8 loads in flight per thread
  static_assert(SCAN <= PF_QUEUE, "a batch never overflows an empty queue");
  for (int base = q_lo; base < q_hi && !fail;) {
    // queue the hot chunks of as many batches as the queue surely holds
    // (usually the CTA's whole range: hot chunks are rare), then test them
    do {
      const int end = min(q_hi, base + SCAN);
      uint32_t sv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + u * NT + tid;
        sv[u] = i < end ? __ldg(Sg + i) : 0u;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (sv[u] >= tau) {
          const int slot = atomicAdd(&s_nq, 1);
          if (slot < PF_QUEUE) queue[slot] = base + u * NT + tid;
        }
      }
      base += SCAN;
      __syncthreads();
    } while (base < q_hi && s_nq + SCAN <= PF_QUEUE);
    const int nq = s_nq;
#if LD_PF_STATS
    if (tid == 0) st_hot += nq;
#endif
    // 2a: each hot chunk's cells >= tau through the neighbour prefilter
    for (int qi = warp; qi < nq; qi += NW) {
      const int64_t w0 = static_cast<int64_t>((c0 + queue[qi]) * SEG_BYTES -
                                              reinterpret_cast<uintptr_t>(A)) / 4;
      constexpr int STEPS = SEG_BYTES / 128;
      uint32_t vv[STEPS];
#pragma unroll
      for (int step = 0; step < STEPS; ++step) {
        const int64_t c = w0 + step * 32 + lane;
        vv[step] = (c >= 0 && c < ncells) ? __ldg(A + c) : 0u;
      }
#pragma unroll
      for (int step = 0; step < STEPS; ++step) {
        const uint32_t v = vv[step];
        const int64_t cell = w0 + step * 32 + lane;
        if (v >= tau && cell >= rc0 && cell < rc1) {
          const int t = static_cast<int>(cell / n_rho);
          const int r = static_cast<int>(cell - static_cast<int64_t>(t) * n_rho);
          const u64 key = mk_key(v, static_cast<uint32_t>(cell));
          if (beats_neighbours(A, n_theta, n_rho, t, r, v, ht, hr)) {
            const int pos = find_desc(keys, nv, key);
            if (pos < 0 || !((s_vbits[pos >> 5] >> (pos & 31)) & 1u)) {
              const int slot = atomicAdd(&s_nsurv, 1);
              if (slot < PF_SURV) surv[slot] = key;
            }
          }
        }
      }
    }
    __syncthreads();
    const int ns = s_nsurv;
    if (ns > PF_SURV) {
      fail = true;
      break;
    }
#if LD_PF_STATS
    if (tid == 0) st_surv += ns;
#endif
    // 2b: the survivors through the exact test, each by a team of T warps
    // (few survivors: the whole CTA shares their windows' rows; many: one
    // warp each), results combined in shared memory
    int T = 1;
    while (T < NW && T * 2 * ns <= NW) T *= 2;
    if (T == 1) {  // a warp per survivor, no barrier between them
      for (int si = warp; si < ns; si += NW) {
        const u64 key = surv[si];
        const uint32_t v = static_cast<uint32_t>(key >> 32);
        const uint32_t idx = 0xFFFFFFFFu - static_cast<uint32_t>(key);
        const int t = static_cast<int>(idx / static_cast<uint32_t>(n_rho));
        const int r = static_cast<int>(idx - static_cast<uint32_t>(t) * n_rho);
        if (warp_window_max<WU, true>(A, ncells, n_theta, n_rho, t, r, v, ht, hr, lane) &&
            lane == 0) {
          const int slot = atomicAdd(ncand0, 1);
          if (slot < SP_CAP) cand0[slot] = key;
        }
      }
      __syncthreads();
    } else {
      const int per = NW / T;  // survivors per round (one round: ns <= per)
      for (int sb = 0; sb < ns; sb += per) {
        const int si = sb + warp / T, part = warp % T;
        bool ok = true;
        if (si < ns) {
          const u64 key = surv[si];
          const uint32_t v = static_cast<uint32_t>(key >> 32);
          const uint32_t idx = 0xFFFFFFFFu - static_cast<uint32_t>(key);
          const int t = static_cast<int>(idx / static_cast<uint32_t>(n_rho));
          const int r = static_cast<int>(idx - static_cast<uint32_t>(t) * n_rho);
          ok = warp_window_max<WU, true>(A, ncells, n_theta, n_rho, t, r, v, ht, hr, lane, part, T);
        }
        if (lane == 0) s_pok[warp] = ok ? 1 : 0;
        __syncthreads();
        if (tid < per && sb + tid < ns) {
          bool all = true;
          for (int j = 0; j < T; ++j) all = all && s_pok[tid * T + j];
          if (all) {
            const int slot = atomicAdd(ncand0, 1);
            if (slot < SP_CAP) cand0[slot] = surv[sb + tid];
          }
        }
        __syncthreads();
      }
    }
    if (tid == 0) {
      s_nq = 0;
      s_nsurv = 0;
    }
    __syncthreads();
  }
  if (fail && tid == 0) atomicOr(fail0, 1);
  pf_sync<G>();  // every candidate and failure in CTA 0
  if (rank != 0) return;
  const int nc = s_ncand;
#if LD_PF_STATS
  st_t3 = clock64();
  if (tid == 0 && p.diag) {
    unsigned long long *o = p.diag + static_cast<int64_t>(f) * PF_DIAG;
    o[0] = st_t1 - st_t0;
    o[1] = st_t2 - st_t1;
    o[2] = st_t3 - st_t2;
    o[3] = st_hot;
    o[4] = st_surv;
    o[5] = nc;
    o[6] = st_rounds;
    o[7] = n_src;
    o[8] = tau_f;
    o[9] = st_tl - st_t0;
    o[10] = st_lat;
    o[11] = st_win;
  }
#endif
  if (s_fail || nc > SP_CAP || nc < p.k) {  // (nc >= k always holds with a certified bound)
    if (tid == 0) {
      p.gtau[f] = tau_f;
      p.resolved[f] = 0u;
    }
    return;
  }

  // ---- 3. the best k of the candidates
  int nc2 = 32;
  while (nc2 < nc) nc2 <<= 1;
  {
    u64 x[SP_CAP / NT];
#pragma unroll
    for (int s = 0; s < SP_CAP / NT; ++s) {
      const int i = s * NT + tid;
      x[s] = i < nc ? cand[i] : 0ull;
    }
    block_sort_desc<NT, SP_CAP / NT>(cand, nc2, x);
  }
  ld_peak *out = p.peaks + static_cast<int64_t>(f) * p.k;
  for (int i = tid; i < p.k; i += NT) {
    const u64 key = cand[i];
    const uint32_t idx = 0xFFFFFFFFu - static_cast<uint32_t>(key);
    ld_peak pk;
    pk.theta_bin = static_cast<int32_t>(idx / static_cast<uint32_t>(n_rho)) + p.theta_offset;
    pk.rho_bin = static_cast<int32_t>(idx % static_cast<uint32_t>(n_rho));
    pk.votes = static_cast<uint32_t>(key >> 32);
    out[i] = pk;
  }
  if (tid == 0) {
    p.n_peaks[f] = p.k;
    p.gtau[f] = tau_f;
    p.resolved[f] = 1u;
  }
}

// ---------------------------------------------------------------------------
// Peak hint from an existing accumulator (ld_hough_hint_from_acc): what the
// voting kernel records while a band is in shared memory (R25, R30), computed
// by one read of the accumulator -- for accumulators that did not come
// straight out of one ld_hough_accumulate_hint call (a sum of partial
// accumulators after an all_reduce, a theta shard voted with a slice of the
// table).  One warp per 1 KB chunk q of a frame's memory: the chunk maximum
// (exact, written once: no atomics), and the best cell (count << 32 | ~cell)
// among the chunk's counters in candidate rows [cand_t0, cand_t1), folded by
// atomicMax into the key of its group of gc consecutive chunks (gc such that
// the keys fit the hint's capacity of n_theta * HINT_MAX_RANGES per frame;
// the host zeroes the keys first).  Header: n_bands * HINT_MAX_RANGES keys.
// ---------------------------------------------------------------------------
struct HintFromAccParams {
  const uint32_t *acc;
  int32_t batch, n_theta, n_rho, cand_t0, cand_t1, n_seg, gc, n_bands;
  uint32_t *hdr;
  unsigned long long *keys;  // [batch][n_bands * HINT_MAX_RANGES]
  uint32_t *segmax;          // [batch][n_seg]
};

constexpr int HF_WARPS = 8;

#ifndef LD_HF_MINB
#define LD_HF_MINB 4  // CTAs per SM the register budget is sized for (1 or 8: slower)
#endif
#ifndef LD_HF_CH
#define LD_HF_CH 4  // chunks per warp in flight
#endif
__global__ void __launch_bounds__(32 * HF_WARPS, LD_HF_MINB) hint_from_acc_kernel(const HintFromAccParams p) {
  LD_PDL_TRIGGER();
  pdl_wait();  // the previous kernel of the stream (acc, hint, flags) is complete
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, f = blockIdx.y;
  if (f == 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    uint32_t *h = p.hdr;
    h[0] = HINT_MAGIC;
    h[1] = static_cast<uint32_t>(p.batch);
    h[2] = static_cast<uint32_t>(p.n_theta);
    h[3] = static_cast<uint32_t>(p.n_rho);
    h[4] = static_cast<uint32_t>(p.n_bands);
    h[5] = static_cast<uint32_t>(HINT_MAX_RANGES);
    h[6] = static_cast<uint32_t>(p.n_seg);
    const uint64_t a = reinterpret_cast<uintptr_t>(p.acc);
    h[7] = static_cast<uint32_t>(a);
    h[8] = static_cast<uint32_t>(a >> 32);
  }
  const int64_t ncells = static_cast<int64_t>(p.n_theta) * p.n_rho;
  const uint32_t *A = p.acc + static_cast<int64_t>(f) * ncells;
  const uintptr_t c0 = reinterpret_cast<uintptr_t>(A) / SEG_BYTES;
  const int64_t r0 = static_cast<int64_t>(p.cand_t0) * p.n_rho, r1 = static_cast<int64_t>(p.cand_t1) * p.n_rho;
  // a chunk is 1 KB-aligned: lane l reads its counters 4l .. 4l+3 and
  // 128+4l .. 131+4l as two 16-byte vectors; the frame's first and last
  // chunks (bytes outside the frame) are read counter by counter
  constexpr int CH = LD_HF_CH;  // chunks per warp in flight
  const int stride = gridDim.x * HF_WARPS;
  for (int q0 = blockIdx.x * HF_WARPS + warp; q0 < p.n_seg; q0 += CH * stride) {
    uint4 v[CH][2];
    int64_t w0[CH];
#pragma unroll
    for (int h = 0; h < CH; ++h) {
      const int q = q0 + h * stride;
      w0[h] = static_cast<int64_t>((c0 + q) * SEG_BYTES - reinterpret_cast<uintptr_t>(A)) / 4;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int64_t c = w0[h] + 128 * j + 4 * lane;
        if (q >= p.n_seg) {
          v[h][j] = make_uint4(0u, 0u, 0u, 0u);
        } else if (w0[h] >= 0 && w0[h] + 256 <= ncells) {
          v[h][j] = __ldg(reinterpret_cast<const uint4 *>(A + c));
        } else {
          v[h][j].x = c + 0 >= 0 && c + 0 < ncells ? __ldg(A + c + 0) : 0u;
          v[h][j].y = c + 1 >= 0 && c + 1 < ncells ? __ldg(A + c + 1) : 0u;
          v[h][j].z = c + 2 >= 0 && c + 2 < ncells ? __ldg(A + c + 2) : 0u;
          v[h][j].w = c + 3 >= 0 && c + 3 < ncells ? __ldg(A + c + 3) : 0u;
        }
      }
    }
#pragma unroll
    for (int h = 0; h < CH; ++h) {
      const int q = q0 + h * stride;
      if (q >= p.n_seg) break;  // warp-uniform
      // the chunk maximum, and the lane's first (lowest-index) maximum among
      // the candidate rows' counters
      uint32_t m = 0u, lm = 0u;
      int64_t li = 0;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const uint32_t e4[4] = {v[h][j].x, v[h][j].y, v[h][j].z, v[h][j].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int64_t c = w0[h] + 128 * j + 4 * lane + e;
          m = max(m, e4[e]);
          if (e4[e] > lm && c >= r0 && c < r1) {
            lm = e4[e];
            li = c;
          }
        }
      }
      m = __reduce_max_sync(0xffffffffu, m);
      u64 best = lm ? mk_key(lm, static_cast<uint32_t>(li)) : 0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const u64 other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other > best ? other : best;
      }
      if (lane == 0) {
        p.segmax[static_cast<int64_t>(f) * p.n_seg + q] = m;
        if (best)
          atomicMax(p.keys + static_cast<int64_t>(f) * p.n_bands * HINT_MAX_RANGES + q / p.gc, best);
      }
    }
  }
}

// keys and chunk groups of the hint of an n_theta x n_rho accumulator
static void hint_geometry(int n_theta, int n_rho, int *n_seg, int *gc, int *n_bands) {
  *n_seg = seg_count(static_cast<int64_t>(n_theta) * n_rho);
  const int64_t cap = static_cast<int64_t>(n_theta) * HINT_MAX_RANGES;  // keys per frame
  *gc = static_cast<int>((*n_seg + cap - 1) / cap);
  const int n_keys = (*n_seg + *gc - 1) / *gc;
  *n_bands = (n_keys + HINT_MAX_RANGES - 1) / HINT_MAX_RANGES;  // <= n_theta
}

size_t hint_self_keys_bytes(int batch, int n_theta, int n_rho) {
  int n_seg, gc, n_bands;
  hint_geometry(n_theta, n_rho, &n_seg, &gc, &n_bands);
  return sizeof(u64) * static_cast<size_t>(batch) * n_bands * HINT_MAX_RANGES;
}

cudaError_t launch_hint_from_acc(const uint32_t *acc, int batch, int n_theta, int n_rho,
                                 int cand_t0, int cand_t1, uint32_t *hdr,
                                 unsigned long long *keys, uint32_t *segmax, cudaStream_t stream) {
  HintFromAccParams p;
  p.acc = acc;
  p.batch = batch;
  p.n_theta = n_theta;
  p.n_rho = n_rho;
  p.cand_t0 = cand_t0;
  p.cand_t1 = cand_t1;
  hint_geometry(n_theta, n_rho, &p.n_seg, &p.gc, &p.n_bands);
  p.hdr = hdr;
  p.keys = keys;
  p.segmax = segmax;
  cudaError_t e = cudaMemsetAsync(p.keys, 0,
                                  sizeof(u64) * static_cast<size_t>(batch) * p.n_bands * HINT_MAX_RANGES,
                                  stream);
  if (e != cudaSuccess) return e;
  // about 8 CTAs per SM over the whole batch, every warp looping over chunks
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int want = (8 * sms + batch - 1) / batch;
  const int gx = std::max(1, std::min(want, (p.n_seg + HF_WARPS - 1) / HF_WARPS));
  dim3 grid(static_cast<unsigned>(gx), batch);
  return launch_ex(hint_from_acc_kernel, grid, dim3(32 * HF_WARPS), 0, stream, 1, p);
}

__global__ void __launch_bounds__(PK_THREADS) peaks_merge_kernel(const PeaksParams p) {
  LD_PDL_TRIGGER();
  pdl_wait();  // the previous kernel of the stream (acc, hint, flags) is complete
  __shared__ u64 buf[PK_BUF];
  __shared__ u64 top[LD_MAX_K];
  __shared__ int s_ntop;
  const int f = blockIdx.x;
  if (frame_resolved(p, f)) return;
  const u64 *in = p.band_keys + static_cast<int64_t>(f) * p.n_units * p.k;
  const int n_in = p.n_units * p.k;
  __shared__ int s_nbuf;
  if (threadIdx.x == 0) {
    s_ntop = 0;
    s_nbuf = 0;
  }
  __syncthreads();
  for (int base = 0; base < n_in; base += PK_CHUNK) {
    // keys not above the current k-th best cannot enter the top-k: skip them
    const u64 kth = (s_ntop == p.k) ? top[p.k - 1] : 0ull;
    const int nb = min(PK_CHUNK, n_in - base);
    for (int i = threadIdx.x; i < nb; i += PK_THREADS) {
      const u64 key = in[base + i];
      if (key > kth) buf[atomicAdd(&s_nbuf, 1)] = key;
    }
    __syncthreads();
    const int n = s_nbuf;
    if (n > 0) {
      merge_topk(buf, n, top, &s_ntop, p.k);
      if (threadIdx.x == 0) s_nbuf = 0;
      __syncthreads();
    }
  }
  const int ntop = s_ntop;
  ld_peak *out = p.peaks + static_cast<int64_t>(f) * p.k;
  int nz = 0;
  for (int i = threadIdx.x; i < p.k; i += PK_THREADS) {
    const u64 key = i < ntop ? top[i] : 0ull;
    ld_peak pk;
    if (key >= (1ull << 32)) {
      const uint32_t idx = 0xFFFFFFFFu - static_cast<uint32_t>(key);
      pk.theta_bin = static_cast<int32_t>(idx / static_cast<uint32_t>(p.n_rho));
      pk.rho_bin = static_cast<int32_t>(idx % static_cast<uint32_t>(p.n_rho));
      pk.votes = static_cast<uint32_t>(key >> 32);
      ++nz;
    } else {
      pk.theta_bin = -1;
      pk.rho_bin = -1;
      pk.votes = 0u;
    }
    out[i] = pk;
  }
  __shared__ int s_nz;
  if (threadIdx.x == 0) s_nz = 0;
  __syncthreads();
  if (nz) atomicAdd(&s_nz, nz);
  __syncthreads();
  if (threadIdx.x == 0) p.n_peaks[f] = s_nz;
}

// ---------------------------------------------------------------------------
// Tiled kernel (the fast path).  CTA = PT_TR theta rows x tc rho columns of one
// frame, blockDim = tch = tc + 2*half_rho loaded columns, HT = half_theta as a
// template parameter so the column (theta-direction) maximum is computed in
// registers with static indexing:
//   1. thread j loads column c0 - hr + j for rows t0-HT .. t0+TR+HT (coalesced
//      across threads), outside the accumulator = 0 (never a candidate, never
//      beats a candidate, never ties one because candidates have votes >= 1);
//   2. Cs[i][j] = max over the 2HT+1 rows around row i (theta window);
//   3. owned cell (i, j) with v >= floor is a window maximum iff
//      v >= Cs[i][j-hr .. j+hr].  A branch-free prefilter (v == Cs[i][j] and
//      v >= Cs[i][j +- 1..2]) keeps ~1/25 of the cells of a noisy
//      accumulator; the survivors are compacted with warp ballots and only
//      they run the full test (nearest-first, early exit);
//   4. a window maximum is a candidate iff no equal value sits at a lower
//      (theta, rho) index inside its window (exact tie-break); only columns
//      whose theta-window maximum equals v can hold such a value, and only
//      those are scanned (the value tile Vs is kept in shared memory);
//   5. candidates (at most one per (HT+1) x (hr+1) block of the tile, so the
//      buffer is sized exactly) are sorted and the tile's best k written out.
// ---------------------------------------------------------------------------
template <int HT>
__global__ void __launch_bounds__(PT_MAX_THREADS) peaks_tile_kernel(const PeaksParams p) {
  LD_PDL_TRIGGER();
  pdl_wait();  // the previous kernel of the stream (acc, hint, flags) is complete
  extern __shared__ __align__(16) unsigned char psm[];
  constexpr int NV = PT_TR + 2 * HT;
  constexpr int PF = 2;  // prefilter radius in rho
  const int tch = p.tch;
  uint32_t *Vs = reinterpret_cast<uint32_t *>(psm);   // [NV][tch] values
  uint32_t *Cs = Vs + NV * tch;                        // [PT_TR][tch] theta-window max
  uint16_t *surv = reinterpret_cast<uint16_t *>(Cs + PT_TR * tch);  // [PT_TR*tch]
  u64 *buf = reinterpret_cast<u64 *>(
      psm + (((NV + PT_TR) * tch * 4 + PT_TR * tch * 2 + 15) & ~15));
  __shared__ int s_nbuf, s_nsurv;

  const int tile = blockIdx.x, f = blockIdx.y;
  if (frame_resolved(p, f)) return;
  const int tt = tile / p.tiles_r, tr = tile - tt * p.tiles_r;
  const int t0 = tt * PT_TR;
  const int hr = p.half_rho;
  const int j = threadIdx.x;
  const int lane = j & 31;
  const int c = tr * p.tc - hr + j;  // global rho column of this thread
  const int n_rho = p.n_rho;

  // ---- phase A: column values (registers + smem) and theta-window maxima
  uint32_t v[NV];
  {
    const bool cin = c >= 0 && c < n_rho;
    const uint32_t *col = p.acc + (static_cast<int64_t>(f) * p.n_theta + (t0 - HT)) * n_rho + c;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int t = t0 - HT + q;
      v[q] = (cin && t >= 0 && t < p.n_theta) ? __ldg(col + static_cast<int64_t>(q) * n_rho) : 0u;
    }
  }
  uint32_t cm[PT_TR];
#pragma unroll
  for (int q = 0; q < NV; ++q) Vs[q * tch + j] = v[q];
#pragma unroll
  for (int i = 0; i < PT_TR; ++i) {
    uint32_t m = v[i];
#pragma unroll
    for (int k = 1; k <= 2 * HT; ++k) m = max(m, v[i + k]);
    cm[i] = m;
    Cs[i * tch + j] = m;
  }
  if (j == 0) {
    s_nbuf = 0;
    s_nsurv = 0;
  }
  __syncthreads();

  // ---- phase B: branch-free prefilter, survivors compacted with warp ballots.
  // A candidate is the maximum of its window, so in particular of its own
  // theta-window column (v == cm) and of the columns within PF.
  const bool owned = j >= hr && j < hr + p.tc && c < n_rho;
  const int pf = hr < PF ? hr : PF;
#pragma unroll
  for (int i = 0; i < PT_TR; ++i) {
    const uint32_t vv = v[i + HT];
    bool pass = owned && (t0 + i < p.n_theta) && vv >= p.floor_votes && vv == cm[i];
    const uint32_t *crow = Cs + i * tch + j;
#pragma unroll
    for (int d = 1; d <= PF; ++d)
      if (d <= pf) pass = pass && crow[owned ? -d : 0] <= vv && crow[owned ? d : 0] <= vv;
    const uint32_t bal = __ballot_sync(0xffffffffu, pass);
    if (bal) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&s_nsurv, __popc(bal));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (pass) surv[base + __popc(bal & ((1u << lane) - 1u))] = static_cast<uint16_t>(i * tch + j);
    }
  }
  __syncthreads();

  // ---- phase C: exact window test for the survivors
  const int nsurv = s_nsurv;
  for (int s = threadIdx.x; s < nsurv; s += blockDim.x) {
    const int idx = surv[s];
    const int i = idx / tch, jj = idx - i * tch;
    const uint32_t vv = Vs[(i + HT) * tch + jj];
    const uint32_t *crow = Cs + i * tch + jj;
    bool ok = true;
    // own column: an equal value in an earlier row of the window
#pragma unroll
    for (int k = 0; k < HT; ++k) ok = ok && Vs[(i + k) * tch + jj] != vv;
    for (int d = 1; ok && d <= hr; ++d) {
      const uint32_t cl = crow[-d], cr = crow[d];
      ok = (cl <= vv) && (cr <= vv);
      if (ok && cl == vv) {  // equal value to the left: lower index in rows t-HT .. t
        for (int q = i; q <= i + HT && ok; ++q) ok = Vs[q * tch + jj - d] != vv;
      }
      if (ok && cr == vv) {  // equal value to the right: lower index in rows t-HT .. t-1
        for (int q = i; q < i + HT && ok; ++q) ok = Vs[q * tch + jj + d] != vv;
      }
    }
    if (ok) {
      const int t = t0 + i;
      const int cc = tr * p.tc - hr + jj;
      buf[atomicAdd(&s_nbuf, 1)] = mk_key(vv, static_cast<uint32_t>(t * n_rho + cc));
    }
  }
  __syncthreads();
  const int n = s_nbuf;
  u64 *out = p.band_keys + (static_cast<int64_t>(f) * p.n_units + tile) * p.k;
  if (n > p.k) {
    int np2 = 1;
    while (np2 < n) np2 <<= 1;
    for (int i = n + threadIdx.x; i < np2; i += blockDim.x) buf[i] = 0ull;
    __syncthreads();
    bitonic_desc(buf, np2);
  }
  for (int i = threadIdx.x; i < p.k; i += blockDim.x) out[i] = i < n ? buf[i] : 0ull;
}


// ---------------------------------------------------------------------------
// Streaming kernel (the fast path, half_theta <= 12).  CTA = one rho strip of
// st_sw owned columns x one chunk of st_tb theta rows of one frame; each of
// the st_nt threads owns CPT columns (c0 - hr + tid + q*st_nt, coalesced),
// streamed down the chunk's rows G at a time with the 2HT rows above kept in
// registers, so every accumulator value is read from HBM once (plus the
// 2HT-row chunk halo) and the theta-window column maximum costs 2HT register
// max operations per cell.  Per candidate row: column maxima -> shared
// memory; a cell can only be a window maximum if it equals its own column
// maximum, and only matters if its votes reach the CTA's running k-th best
// candidate (tau): such cells -- few -- scan the +-hr column maxima, then
// resolve exact ties (equal values at a lower (theta, rho) index) from the
// accumulator itself.  Candidates are merged into the CTA's top-k in shared
// memory; peaks_merge_kernel merges the CTAs of a frame.
// ---------------------------------------------------------------------------
constexpr int PS_G = 4;    // rows per register group
constexpr int PS_NPF = 2;  // groups of L2 prefetch beyond the register prefetch

constexpr int PS_NT_MAX = 512;   // threads per CTA, one CTA per SM
constexpr int PS_NT_MAX2 = 384;  // threads per CTA when two CTAs share an SM
// register window (2 groups + 2HT rows) x CPT small enough for two CTAs per SM
#ifndef LD_PS_MINB_LIMIT
#define LD_PS_MINB_LIMIT 48
#endif
constexpr int ps_minb(int ht, int cpt) { return (2 * PS_G + 2 * ht) * cpt <= LD_PS_MINB_LIMIT ? 2 : 1; }

template <int CPT>
__device__ __forceinline__ void stream_store(uint32_t *dst, const uint32_t (&v)[CPT]) {
  if constexpr (CPT == 4) {
    *reinterpret_cast<uint4 *>(dst) = make_uint4(v[0], v[1], v[2], v[3]);
  } else if constexpr (CPT == 2) {
    *reinterpret_cast<uint2 *>(dst) = make_uint2(v[0], v[1]);
  } else {
#pragma unroll
    for (int q = 0; q < CPT; ++q) dst[q] = v[q];
  }
}

// CTA = st_nt threads x CPT consecutive columns each; rows are read with
// plain coalesced loads through a per-thread row pointer (immediate column
// offsets), one group of PS_G rows ahead of the group being tested (register
// double buffering), so HBM latency overlaps the arithmetic.  Columns outside
// the accumulator are read through a clamped pointer and masked to 0.
template <int HT, int CPT, int MINB>
__global__ void __launch_bounds__(MINB == 2 ? PS_NT_MAX2 : PS_NT_MAX, MINB)
    peaks_stream_kernel(const PeaksParams p) {
  LD_PDL_TRIGGER();
  pdl_wait();  // the previous kernel of the stream (acc, hint, flags) is complete
  constexpr int NV = PS_G + 2 * HT;
  static_assert(PS_G * CPT <= 32, "survivor mask");
  extern __shared__ __align__(16) unsigned char psm[];
  const int nt = p.st_nt;
  const int width = nt * CPT;                          // loaded columns
  uint32_t *CM = reinterpret_cast<uint32_t *>(psm);     // [PS_G][width] column maxima
  u64 *top = reinterpret_cast<u64 *>(CM + PS_G * width);  // [k] (8-aligned: width even)
  u64 *buf = top + p.k;                                 // [pow2(candidate bound + k)]
  uint32_t *SL = reinterpret_cast<uint32_t *>(buf + p.st_buf);  // [PS_G * sw] survivors
  __shared__ int s_nbuf, s_ntop, s_nsurv;
  __shared__ uint32_t s_tau;

  const int unit = blockIdx.x, f = blockIdx.y;
  if (frame_resolved(p, f)) return;
  const int strip = unit / p.st_chunks, chunk = unit - strip * p.st_chunks;
  const int hr = p.half_rho, n_rho = p.n_rho, n_theta = p.n_theta;
  const int cbase = strip * p.st_sw - hr;  // global column of loaded column 0
  const int tb0 = p.cand_t0 + chunk * p.st_tb;
  const int tb1 = min(tb0 + p.st_tb, p.cand_t1);
  const int tid = threadIdx.x;

  const int j0 = tid * CPT;  // loaded columns j0 .. j0+CPT-1
  const int col0 = cbase + j0;
  const int colc = min(max(col0, 0), n_rho - CPT);  // clamped: every load in bounds
  uint32_t cmask[CPT];
  bool own[CPT];
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int col = col0 + q;
    const bool in = col >= 0 && col < n_rho;
    cmask[q] = in ? 0xFFFFFFFFu : 0u;
    own[q] = in && j0 + q >= hr && j0 + q < hr + p.st_sw;
  }
  const bool shifted = colc != col0;  // edge thread: clamped columns differ
  const bool hr_wide = hr >= 2 * CPT - 1;  // all in-thread and adjacent-thread columns in the window
  if (tid == 0) {
    s_nbuf = 0;
    s_ntop = 0;
    s_nsurv = 0;
    s_tau = p.floor_votes;
  }
  const uint32_t *rowp = p.acc + (static_cast<int64_t>(f) * n_theta + (tb0 - HT)) * n_rho + colc;
  int rnext = tb0 - HT;  // row rowp points at
  auto load_row = [&](uint32_t (&dst)[CPT]) {
    uint32_t t[CPT];
    if (rnext >= 0 && rnext < n_theta) {
#pragma unroll
      for (int q = 0; q < CPT; ++q) t[q] = __ldg(rowp + q);
    } else {
#pragma unroll
      for (int q = 0; q < CPT; ++q) t[q] = 0u;
    }
    if (shifted) {  // edge thread: place clamped columns at their loaded index
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        uint32_t v = 0u;
#pragma unroll
        for (int u = 0; u < CPT; ++u)
          if (colc + u == col0 + q) v = t[u];
        dst[q] = v & cmask[q];
      }
    } else {
#pragma unroll
      for (int q = 0; q < CPT; ++q) dst[q] = t[q];
    }
    rowp += n_rho;
    ++rnext;
  };

  // V[k][q] = row (g0 - HT + k); N[k][q] = next group's new rows
  uint32_t V[NV][CPT], N[PS_G][CPT];
#pragma unroll
  for (int k = 0; k < NV; ++k) load_row(V[k]);
  __syncthreads();

  // L2 prefetch of the strip's row segments PS_NPF groups ahead (one bulk
  // prefetch per row, issued by one thread): the register loads of the next
  // group then hit L2 instead of paying the HBM round trip
  const uint32_t *frame0 = p.acc + static_cast<int64_t>(f) * n_theta * n_rho;
  const uintptr_t acc_end = reinterpret_cast<uintptr_t>(p.acc + static_cast<int64_t>(p.batch) * n_theta * n_rho);
  const int pc0 = max(cbase, 0), pc1 = min(cbase + width, n_rho);
  // rows are spread over the warps (lane 0 of warp w issues row r0 + w, ...)
  // so that no single warp carries the prefetch work into the group barrier
  const bool pf_lane = (tid & 31) == 0;
  const int pf_w = tid >> 5, pf_nw = nt >> 5;
  auto l2_prefetch_rows = [&](int r0, int r1) {
    if (!pf_lane) return;
    for (int r = max(r0, 0) + pf_w; r < min(r1, n_theta); r += pf_nw) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(frame0 + static_cast<int64_t>(r) * n_rho + pc0) & ~static_cast<uintptr_t>(15);
      uintptr_t e = (reinterpret_cast<uintptr_t>(frame0 + static_cast<int64_t>(r) * n_rho + pc1) + 15) & ~static_cast<uintptr_t>(15);
      if (e > (acc_end & ~static_cast<uintptr_t>(15))) e = acc_end & ~static_cast<uintptr_t>(15);
      if (e > a)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(static_cast<uint32_t>(e - a))
                     : "memory");
    }
  };
  l2_prefetch_rows(tb0 + HT + PS_G, tb0 + HT + (1 + PS_NPF) * PS_G);

  for (int g0 = tb0; g0 < tb1; g0 += PS_G) {
    l2_prefetch_rows(g0 + HT + (1 + PS_NPF) * PS_G, g0 + HT + (2 + PS_NPF) * PS_G);
    if (g0 + PS_G < tb1) {
#pragma unroll
      for (int k = 0; k < PS_G; ++k) load_row(N[k]);  // in flight during this group
    }
    // thread 0 prefetches the per-frame threshold now; it is used after the
    // group, so the global round trip overlaps the group's work
    uint32_t gt = 0;
    if (tid == 0) gt = ld_relaxed_u32(p.gtau + f);
    uint32_t tq[CPT];  // per column: tau if owned, else "never"
    const uint32_t tau = s_tau;
#pragma unroll
    for (int q = 0; q < CPT; ++q) tq[q] = own[q] ? tau : 0xFFFFFFFFu;
    const int nrows = min(PS_G, tb1 - g0);
    uint32_t surv = 0;
#pragma unroll
    for (int i = 0; i < PS_G; ++i) {
      // per column: mu = max of the HT rows above, md = of the HT rows below;
      // the cell beats its own column of the window with the tie rule iff
      // v > mu and v >= md (an equal value above has a lower index)
      uint32_t m[CPT], strict = 0;
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        uint32_t mu = 0, md = 0;
#pragma unroll
        for (int k = 0; k < HT; ++k) mu = max(mu, V[i + k][q]);
#pragma unroll
        for (int k = 1; k <= HT; ++k) md = max(md, V[i + HT + k][q]);
        const uint32_t v = V[i + HT][q];
        m[q] = max(max(mu, md), v);
        strict |= static_cast<uint32_t>(v > mu) << q;
      }
      // prefilter: a window maximum is >= the column maxima of every column
      // within +-hr -- here the thread's own CPT columns and the nearest
      // column of each neighbouring thread (when hr reaches them)
      uint32_t hm = 0;
#pragma unroll
      for (int q = 0; q < CPT; ++q) hm = max(hm, m[q]);
      const uint32_t ml = __shfl_up_sync(0xffffffffu, m[CPT - 1], 1);
      const uint32_t mr = __shfl_down_sync(0xffffffffu, m[0], 1);
      if (hr_wide) hm = max(hm, max(ml, mr));  // lanes 0/31 get their own values back
      if (hm >= tau) {  // else no cell of this thread's row can reach tau
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          const uint32_t need = hr_wide ? hm : m[q];
          surv |= static_cast<uint32_t>(V[i + HT][q] >= max(need, tq[q]) && ((strict >> q) & 1u))
                  << (i * CPT + q);
        }
      }
      stream_store(CM + i * width + j0, m);
    }
    if (nrows < PS_G) surv &= (1u << (nrows * CPT)) - 1u;
    while (surv) {  // survivor list of the group: (row << 16) | loaded column
      const int b = __ffs(surv) - 1;
      surv &= surv - 1;
      const int i = b / CPT, q = b - i * CPT;
      const int slot = atomicAdd(&s_nsurv, 1);
      if (LD_CHK(slot < PS_G * p.st_sw))
        SL[slot] = (static_cast<uint32_t>(i) << 16) | static_cast<uint32_t>(j0 + q);
    }
    __syncthreads();  // (1) CM and the survivor list of the group complete
    {
      // one warp per survivor: the lanes scan the +-hr column maxima and the
      // tie rows in parallel (ballots), instead of one divergent lane each
      const int lane = tid & 31, nw = nt >> 5;
      const int nsurv = s_nsurv;
      for (int sidx = tid >> 5; sidx < nsurv; sidx += nw) {
        const uint32_t e = SL[sidx];
        const int i = static_cast<int>(e >> 16), j = static_cast<int>(e & 0xFFFFu);
        const uint32_t *cmr = CM + i * width + j;
        const uint32_t v = *cmr;  // == the cell's own value
        bool bad = false, tie = false;
        for (int d = 1 + lane; d <= hr; d += 32) {
          const uint32_t l = cmr[-d], r = cmr[d];
          bad = bad || l > v || r > v;
          tie = tie || l == v || r == v;
        }
        if (!__any_sync(0xffffffffu, bad) && __any_sync(0xffffffffu, tie)) {
          // equal column maxima: an equal value at a lower (theta, rho) index
          // -- to the left rows up to the cell's own, to the right rows above
          // (re-read from the accumulator: ties are rare)
          const int t = g0 + i;
          for (int d = 1 + lane; d <= hr && !bad; d += 32) {
            if (cmr[-d] == v)
              for (int row = max(t - HT, 0); row <= t && !bad; ++row)
                bad = __ldg(frame0 + static_cast<int64_t>(row) * n_rho + cbase + j - d) == v;
            if (!bad && cmr[d] == v)
              for (int row = max(t - HT, 0); row < t && !bad; ++row)
                bad = __ldg(frame0 + static_cast<int64_t>(row) * n_rho + cbase + j + d) == v;
          }
        }
        if (!__any_sync(0xffffffffu, bad) && lane == 0) {
          const int slot = atomicAdd(&s_nbuf, 1);
          if (LD_CHK(slot < p.st_buf))
            buf[slot] = mk_key(v, static_cast<uint32_t>((g0 + i + p.theta_offset) * n_rho + cbase + j));
        }
      }
    }
    __syncthreads();  // (2) candidates buffered; CM / SL free
    const int nbuf = s_nbuf;
    if (nbuf > 0) merge_topk(buf, nbuf, top, &s_ntop, p.k);
    if (tid == 0) {
      // the frame's k-th best candidate is at least any unit's k-th best:
      // share it through the per-frame threshold
      s_nsurv = 0;
      s_nbuf = 0;
      uint32_t t = s_tau;
      if (nbuf > 0 && s_ntop == p.k) {
        t = max(t, static_cast<uint32_t>(top[p.k - 1] >> 32));
        atomicMax(p.gtau + f, t);  // no return value used: a fire-and-forget RED
      }
      s_tau = max(t, gt);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 2 * HT; ++k)
#pragma unroll
      for (int q = 0; q < CPT; ++q) V[k][q] = V[k + PS_G][q];
#pragma unroll
    for (int k = 0; k < PS_G; ++k)
#pragma unroll
      for (int q = 0; q < CPT; ++q) V[2 * HT + k][q] = N[k][q];
  }
  u64 *out = p.band_keys + (static_cast<int64_t>(f) * p.n_units + unit) * p.k;
  const int ntop = s_ntop;
  for (int i = tid; i < p.k; i += nt) out[i] = i < ntop ? top[i] : 0ull;
}

typedef void (*StreamKernel)(const PeaksParams);
// two CTAs per SM where the register window is small (<= 85 registers)
#define LD_SK(HT, CPT) peaks_stream_kernel<HT, CPT, ps_minb(HT, CPT)>
static StreamKernel stream_kernel(int ht, int cpt) {
  if (cpt == 4) {
    switch (ht) {
      case 0: return LD_SK(0, 4);
      case 1: return LD_SK(1, 4);
      case 2: return LD_SK(2, 4);
      case 3: return LD_SK(3, 4);
      case 4: return LD_SK(4, 4);
      case 5: return LD_SK(5, 4);
      case 6: return LD_SK(6, 4);
      default: return nullptr;
    }
  }
  switch (ht) {
    case 0: return LD_SK(0, 2);
    case 1: return LD_SK(1, 2);
    case 2: return LD_SK(2, 2);
    case 3: return LD_SK(3, 2);
    case 4: return LD_SK(4, 2);
    case 5: return LD_SK(5, 2);
    case 6: return LD_SK(6, 2);
    case 7: return LD_SK(7, 2);
    case 8: return LD_SK(8, 2);
    case 9: return LD_SK(9, 2);
    case 10: return LD_SK(10, 2);
    case 11: return LD_SK(11, 2);
    case 12: return LD_SK(12, 2);
    default: return nullptr;
  }
}
#undef LD_SK

static int pow2_ceil(int v) {
  int n = 1;
  while (n < v) n <<= 1;
  return n;
}

// Candidates of one group: two window maxima are never inside each other's
// window, so a PS_G x sw block holds at most one per (ht+1) x (hr+1) cell.
static int stream_buf_entries(int sw, int ht, int hr, int k) {
  const int bound = ((PS_G + ht) / (ht + 1)) * ((sw + hr) / (hr + 1));
  return pow2_ceil(bound + k);
}
static size_t stream_smem_bytes(int width, int sw, int ht, int hr, int k) {
  (void)ht;
  return sizeof(uint32_t) * static_cast<size_t>(PS_G) * width +
         sizeof(u64) * (static_cast<size_t>(k) + stream_buf_entries(sw, ht, hr, k)) +
         sizeof(uint32_t) * static_cast<size_t>(PS_G) * sw;
}

// Streaming geometry: strips x chunks minimising loaded columns, with enough
// CTAs to fill the GPU.  Returns false when the generic band kernel must run.
static bool peaks_stream_plan(int batch, int n_theta, int n_rho, int half_theta, int half_rho,
                              int k, int sm_count, PeaksParams *p, int *cpt_out, size_t *smem) {
  if (half_theta > PT_MAX_HT) return false;
  int cpt = half_theta <= LD_PS_CPT4_MAX_HT ? 4 : 2;
  if (n_rho < cpt) cpt = 2;      // the clamped row pointer needs n_rho >= CPT
  if (n_rho < cpt) return false;  // (n_rho = 2D + 1 >= 3 for every image)
  int best_s = 0, best_nt = 0;
  long best_cost = -1;
  for (int s = 1; s <= 4096; ++s) {
    const int sw = (n_rho + s - 1) / s;
    if (sw < 32 && s > 1) break;
    const int need = sw + 2 * half_rho;
    const int nt = (((need + cpt - 1) / cpt) + 31) / 32 * 32;
    if (nt > (ps_minb(half_theta, cpt) == 2 ? PS_NT_MAX2 : PS_NT_MAX)) continue;
    const size_t sm_bytes = stream_smem_bytes(nt * cpt, sw, half_theta, half_rho, k);
    if (sm_bytes > 220 * 1024) continue;
    const long cost = static_cast<long>(s) * nt * cpt;
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best_s = s;
      best_nt = nt;
    }
    if (best_cost >= 0 && static_cast<long>(s) * 32 * cpt > 2 * best_cost) break;
  }
  if (!best_s) return false;
  const int sw = (n_rho + best_s - 1) / best_s;
  // theta chunks: enough CTAs to fill the GPU, with the best wave quantisation
  // (CTAs per SM from the kernel variant; each chunk re-reads a
  // 2*half_theta-row halo)
  const int slots = sm_count * ps_minb(half_theta, cpt);
  int chunks = 1;
  double best_eff = -1.0;
  for (int c = 1; c <= 64; ++c) {
    int tbc = (n_theta + c - 1) / c;
    tbc = ((tbc + PS_G - 1) / PS_G) * PS_G;
    if (tbc < 16 && c > 1) break;
    const int cc = (n_theta + tbc - 1) / tbc;
    const long units = static_cast<long>(batch) * best_s * cc;
    const long waves = (units + slots - 1) / slots;
    const double eff = static_cast<double>(units) / (waves * slots) *
                       static_cast<double>(tbc) / (tbc + 2 * half_theta);
    if (eff > best_eff + 1e-3) {
      best_eff = eff;
      chunks = cc;
    }
  }
  int tb = (n_theta + chunks - 1) / chunks;
  tb = ((tb + PS_G - 1) / PS_G) * PS_G;
  if (tb < 16) tb = 16;
  chunks = (n_theta + tb - 1) / tb;
  const size_t bytes = stream_smem_bytes(best_nt * cpt, sw, half_theta, half_rho, k);
  if (bytes > 220 * 1024) return false;
  p->st_buf = stream_buf_entries(sw, half_theta, half_rho, k);
  p->st_nt = best_nt;
  p->st_sw = sw;
  p->st_strips = best_s;
  p->st_tb = tb;
  p->st_chunks = chunks;
  p->n_units = best_s * chunks;
  *cpt_out = cpt;
  *smem = bytes;
  return true;
}


// ---------------------------------------------------------------------------
// Warp-strip kernel (narrow windows: half_theta <= 3, 4 <= half_rho <= 64,
// k <= 64).  Every WARP is an independent unit: one strip of 256 loaded
// columns (owned: 256 - 2 half_rho) x one chunk of theta rows of one frame,
// 8 lane-strided columns per lane (each load instruction reads 32 consecutive
// words).  Nothing is shared between warps, so there is no CTA barrier: the
// latency of one warp's loads is hidden by the other warps.  (Measured on
// B200, tools/stream_probe.cu: this pattern streams at ~5.8 TB/s; per-warp
// cp.async.bulk row copies into a shared ring only reach ~2.6 TB/s.)
//
// Rows stream through a register ring of R = 2 PW_G + 2 HT rows; the row loop
// is unrolled over one ring period, so every ring index is a compile-time
// constant and no register is ever copied.  Per cell, in registers: the
// maximum of the HT rows above (mu) and of the HT rows below (md); the cell
// survives iff v > mu, v >= md and v >= tau -- i.e. it beats its own column
// of the window with the lowest-(theta, rho) tie rule already applied (an
// equal value above has a lower index, one below a higher one).  A group
// whose centre values are all below tau (the running k-th best candidate of
// the warp, raised by the per-frame threshold other warps publish) costs only
// its loads and one max per cell.  The per-frame threshold is polled once per
// ring period and used one period later, so its round trip never stalls the
// warp.  Survivors are
// tested against the column maxima of the +-half_rho neighbouring columns
// (pw_survivors, out of line to keep the unrolled loop small): in-lane +-2
// prefilter, then a warp-cooperative scan; an equal neighbouring maximum is
// resolved exactly from the frame.
// ---------------------------------------------------------------------------
constexpr int PW_CPT = 8, PW_G = 2, PW_W = 8, PW_COLS = 32 * PW_CPT, PW_KMAX = 64, PW_CBUF = 128;

struct PwSmem {
  uint32_t CM[PW_G][PW_COLS];  // column maxima of the group's rows (when a survivor exists)
  u64 top[PW_KMAX];            // the warp's top-k, descending
  u64 cbuf[PW_CBUF];           // candidates of the group
};

struct PwState {
  int ntop;
  uint32_t gt;
};

// The rare path of the warp-strip kernel, kept out of its unrolled row loop
// (instruction-cache footprint): exact +-hr test of the group's survivors
// against the column maxima in S.CM, tie resolution from the frame, insertion
// into the warp's top-k and publication of the k-th best value.  `gt` is the
// warp's threshold on entry; the returned one includes the warp's own k-th
// best (warp-uniform).
template <int HT>
__device__ __noinline__ PwState pw_survivors(PwSmem &S, uint32_t surv, int lane, int g0, int hr,
                                             int cbase, const uint32_t *frame, int n_rho, int k,
                                             int theta_offset, uint32_t *gtau_f, int ntop,
                                             uint32_t gt) {
  {  // per-lane prefilter on the nearest column maxima
    uint32_t t = surv;
    while (t) {
      const int b = __ffs(t) - 1;
      t &= t - 1u;
      const int i = b / PW_CPT, q = b - i * PW_CPT;
      const int j = lane + 32 * q;
      const uint32_t v = S.CM[i][j];
      bool ok = true;
#pragma unroll
      for (int d = 1; d <= 2; ++d) ok = ok && S.CM[i][j - d] <= v && S.CM[i][j + d] <= v;
      if (!ok) surv &= ~(1u << b);
    }
  }
  int ncand = 0;
  for (;;) {  // warp-cooperative exact test of each remaining survivor
    const uint32_t bal = __ballot_sync(0xffffffffu, surv != 0u);
    if (!bal) break;
    const int src = __ffs(bal) - 1;
    const int b = __shfl_sync(0xffffffffu, __ffs(surv) - 1, src);
    if (lane == src) surv &= surv - 1u;
    const int i = b / PW_CPT, q = b - i * PW_CPT;
    const int j = src + 32 * q;
    const uint32_t *cmr = S.CM[i] + j;
    const uint32_t v = *cmr;
    bool bad = false, tie = false;
    for (int d = 1 + lane; d <= hr; d += 32) {
      const uint32_t l = cmr[-d], r = cmr[d];
      bad = bad || l > v || r > v;
      tie = tie || l == v || r == v;
    }
    if (!__any_sync(0xffffffffu, bad) && __any_sync(0xffffffffu, tie)) {
      // an equal column maximum: reject iff an equal cell has a lower
      // (theta, rho) index -- to the left rows up to the cell's own, to
      // the right rows strictly above (values re-read from the frame)
      const int t = g0 + i;
      for (int d = 1 + lane; d <= hr && !bad; d += 32) {
        if (cmr[-d] == v) {
          const int c = cbase + j - d;
          for (int row = max(t - HT, 0); row <= t && !bad; ++row)
            bad = __ldg(frame + static_cast<int64_t>(row) * n_rho + c) == v;
        }
        if (!bad && cmr[d] == v) {
          const int c = cbase + j + d;
          for (int row = max(t - HT, 0); row < t && !bad; ++row)
            bad = __ldg(frame + static_cast<int64_t>(row) * n_rho + c) == v;
        }
      }
    }
    if (!__any_sync(0xffffffffu, bad)) {
      if (lane == 0 && LD_CHK(ncand < PW_CBUF))
        S.cbuf[ncand] = mk_key(v, static_cast<uint32_t>((g0 + i + theta_offset) * n_rho + cbase + j));
      ++ncand;
    }
  }
  __syncwarp();
  if (lane == 0) {  // insertion into the warp's top-k (candidates are rare)
    for (int c = 0; c < ncand; ++c) {
      const u64 key = S.cbuf[c];
      if (ntop == k && key <= S.top[ntop - 1]) continue;
      int pos = ntop < k ? ntop : k - 1;
      while (pos > 0 && S.top[pos - 1] < key) {
        S.top[pos] = S.top[pos - 1];
        --pos;
      }
      S.top[pos] = key;
      if (ntop < k) ++ntop;
    }
    if (ncand > 0 && ntop == k) {
      const uint32_t kth = static_cast<uint32_t>(S.top[k - 1] >> 32);
      if (kth > gt) atomicMax(gtau_f, kth);
      gt = max(gt, kth);
    }
  }
  ntop = __shfl_sync(0xffffffffu, ntop, 0);
  gt = __shfl_sync(0xffffffffu, gt, 0);
  return PwState{ntop, gt};
}

template <int HT>
#ifndef LD_PW_MINB
#define LD_PW_MINB 2
#endif
__global__ void __launch_bounds__(32 * PW_W, LD_PW_MINB) peaks_warp_kernel(const PeaksParams p) {
  LD_PDL_TRIGGER();
  pdl_wait();  // the previous kernel of the stream (acc, hint, flags) is complete
  extern __shared__ __align__(16) unsigned char psm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x * PW_W + warp, f = blockIdx.y;
  if (frame_resolved(p, f)) return;
  if (unit >= p.n_units) return;  // whole warp; no CTA-wide synchronisation below
  PwSmem &S = reinterpret_cast<PwSmem *>(psm)[warp];
  constexpr int NV = PW_G + 2 * HT;  // rows one group reads
  constexpr int R = NV + PW_G;       // ring: + the next group's rows in flight
  constexpr int U = R / PW_G;        // groups per ring period
  static_assert(R % PW_G == 0, "ring must hold whole groups");
  const int strip = unit / p.st_chunks, chunk = unit - strip * p.st_chunks;
  const int hr = p.half_rho, n_rho = p.n_rho, n_theta = p.n_theta;
  const int cbase = strip * p.st_sw - hr;  // global column of loaded column 0
  const int tb0 = p.cand_t0 + chunk * p.st_tb;
  const int tb1 = min(tb0 + p.st_tb, p.cand_t1);
  const uint32_t *frame = p.acc + static_cast<int64_t>(f) * n_theta * n_rho;
  const bool all_in = cbase >= 0 && cbase + PW_COLS <= n_rho;  // warp-uniform
  uint32_t cinm = 0, ownm = 0;
#pragma unroll
  for (int q = 0; q < PW_CPT; ++q) {
    const int j = lane + 32 * q, col = cbase + j;
    const bool in = col >= 0 && col < n_rho;
    cinm |= static_cast<uint32_t>(in) << q;
    ownm |= static_cast<uint32_t>(in && j >= hr && j < hr + p.st_sw) << q;
  }
  const uint32_t own2 = ownm | (ownm << PW_CPT);
  const uint32_t *rowp = frame + static_cast<int64_t>(tb0 - HT) * n_rho + cbase + lane;
  int rnext = tb0 - HT;
  auto load_row = [&](uint32_t (&dst)[PW_CPT]) {
    if (rnext >= 0 && rnext < n_theta) {
      if (all_in) {
#pragma unroll
        for (int q = 0; q < PW_CPT; ++q) dst[q] = __ldg(rowp + 32 * q);
      } else {
#pragma unroll
        for (int q = 0; q < PW_CPT; ++q) dst[q] = ((cinm >> q) & 1u) ? __ldg(rowp + 32 * q) : 0u;
      }
    } else {
#pragma unroll
      for (int q = 0; q < PW_CPT; ++q) dst[q] = 0u;
    }
    rowp += n_rho;
    ++rnext;
  };

  int ntop = 0;                  // warp-uniform
  uint32_t tau = p.floor_votes;  // warp-uniform
  uint32_t gt_next = 0;          // lane 0: per-frame threshold read last group
  const bool hinted = p.hint_hdr != nullptr && p.cand_t0 == 0 && p.cand_t1 == n_theta &&
                      p.theta_offset == 0;
  if (lane == 0) gt_next = ld_relaxed_u32(p.gtau + f);  // first poll, before the row loads
  uint32_t ring[R][PW_CPT];
#pragma unroll
  for (int k = 0; k < NV; ++k) load_row(ring[k]);

  for (int gp = tb0; gp < tb1; gp += U * PW_G) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int g0 = gp + u * PW_G;
      if (g0 >= tb1) break;  // warp-uniform
#define RG(k) ring[(u * PW_G + (k)) % R]
      if (g0 + PW_G < tb1) {
#pragma unroll
        for (int k = 0; k < PW_G; ++k) load_row(RG(NV + k));
      }
      // poll every group when the threshold must be learned, once per ring
      // period when the peak hint already started it near the k-th best
      // (measured: tools/exp_tau_oracle.py, 0.30 vs 0.36 ms unhinted, 0.16 vs
      // 0.15 ms from the true k-th value)
      if (!hinted || u == 0) {
        // the threshold read one poll ago has arrived; read the next one
        const uint32_t gt = gt_next;
        if (lane == 0) gt_next = ld_relaxed_u32(p.gtau + f);
        tau = max(tau, __shfl_sync(0xffffffffu, gt, 0));
      }
      const int nrows = min(PW_G, tb1 - g0);
      const uint32_t rmask = nrows < PW_G ? ((1u << (nrows * PW_CPT)) - 1u) : 0xFFFFu;
      // quick reject: no centre value of the warp reaches tau
      uint32_t hm = 0;
#pragma unroll
      for (int i = 0; i < PW_G; ++i)
#pragma unroll
        for (int q = 0; q < PW_CPT; ++q) hm = max(hm, RG(i + HT)[q]);
      uint32_t surv = 0;
      if (__any_sync(0xffffffffu, hm >= tau)) {
#pragma unroll
        for (int i = 0; i < PW_G; ++i) {
#pragma unroll
          for (int q = 0; q < PW_CPT; ++q) {
            const uint32_t v = RG(i + HT)[q];
            uint32_t mu = 0, md = tau;
#pragma unroll
            for (int k = 0; k < HT; ++k) mu = max(mu, RG(i + k)[q]);
#pragma unroll
            for (int k = 1; k <= HT; ++k) md = max(md, RG(i + HT + k)[q]);
            surv |= static_cast<uint32_t>(v > mu && v >= md) << (i * PW_CPT + q);
          }
        }
        surv &= own2 & rmask;
      }
      if (__any_sync(0xffffffffu, surv != 0u)) {
        // column maxima of the group for the +-hr neighbour tests
#pragma unroll
        for (int i = 0; i < PW_G; ++i)
#pragma unroll
          for (int q = 0; q < PW_CPT; ++q) {
            uint32_t mm = RG(i)[q];
#pragma unroll
            for (int k = 1; k <= 2 * HT; ++k) mm = max(mm, RG(i + k)[q]);
            S.CM[i][lane + 32 * q] = mm;
          }
        __syncwarp();
        const PwState st = pw_survivors<HT>(S, surv, lane, g0, hr, cbase, frame, n_rho, p.k,
                                            p.theta_offset, p.gtau + f, ntop, tau);
        ntop = st.ntop;
        tau = st.gt;  // the warp's own k-th best, if its list is full (uniform)
      }
#undef RG
    }
  }
  u64 *out = p.band_keys + (static_cast<int64_t>(f) * p.n_units + unit) * p.k;
  for (int i = lane; i < p.k; i += 32) out[i] = i < ntop ? S.top[i] : 0ull;
}

typedef void (*WarpKernel)(const PeaksParams);
static WarpKernel warp_kernel(int ht) {
  switch (ht) {
    case 0: return peaks_warp_kernel<0>;
    case 1: return peaks_warp_kernel<1>;
    case 2: return peaks_warp_kernel<2>;
    case 3: return peaks_warp_kernel<3>;
    default: return nullptr;
  }
}
static size_t warp_smem_bytes(int) { return PW_W * sizeof(PwSmem); }

// Warp-strip geometry; false when the window or k do not fit the kernel.
static bool peaks_warp_plan(int batch, int n_theta, int n_rho, int half_theta, int half_rho, int k,
                            int sm_count, PeaksParams *p, size_t *smem) {
  if (half_theta > 3 || half_rho < 4 || half_rho > 64 || k > PW_KMAX || n_rho < PW_CPT)
    return false;
  const int sw = PW_COLS - 2 * half_rho;
  const int strips = (n_rho + sw - 1) / sw;
  const long slots = 2L * PW_W * sm_count;  // warps resident at once
  int chunks = 1;
  double best = -1.0;
  for (int c = 1; c <= 64; ++c) {
    int tb = (n_theta + c - 1) / c;
    tb = (tb + PW_G - 1) / PW_G * PW_G;
    if (tb < 8 && c > 1) break;
    const int cc = (n_theta + tb - 1) / tb;
    const long units = static_cast<long>(batch) * strips * cc;
    const long waves = (units + slots - 1) / slots;
    const double eff = static_cast<double>(units) / (waves * slots) * tb / (tb + 2.0 * half_theta);
    if (eff > best + 1e-3) {
      best = eff;
      chunks = cc;
    }
  }
  int tb = (n_theta + chunks - 1) / chunks;
  tb = (tb + PW_G - 1) / PW_G * PW_G;
  chunks = (n_theta + tb - 1) / tb;
  // the workspace holds ceil(n_theta/16) * ceil(n_rho/32) unit lists per frame
  const long cap = static_cast<long>((n_theta + PT_TR - 1) / PT_TR) * ((n_rho + 31) / 32);
  if (static_cast<long>(strips) * chunks > cap) return false;
  p->st_sw = sw;
  p->st_strips = strips;
  p->st_tb = tb;
  p->st_chunks = chunks;
  p->n_units = strips * chunks;
  *smem = warp_smem_bytes(half_theta);
  return true;
}

typedef void (*TileKernel)(const PeaksParams);
static TileKernel tile_kernel(int ht) {
  switch (ht) {
    case 0: return peaks_tile_kernel<0>;
    case 1: return peaks_tile_kernel<1>;
    case 2: return peaks_tile_kernel<2>;
    case 3: return peaks_tile_kernel<3>;
    case 4: return peaks_tile_kernel<4>;
    case 5: return peaks_tile_kernel<5>;
    case 6: return peaks_tile_kernel<6>;
    case 7: return peaks_tile_kernel<7>;
    case 8: return peaks_tile_kernel<8>;
    case 9: return peaks_tile_kernel<9>;
    case 10: return peaks_tile_kernel<10>;
    case 11: return peaks_tile_kernel<11>;
    case 12: return peaks_tile_kernel<12>;
    default: return nullptr;
  }
}

// Tile geometry for a window; returns false when the generic band kernel must be used.
static bool peaks_tile_plan(int n_theta, int n_rho, int half_theta, int half_rho, int k, PeaksParams *p,
                     size_t *smem) {
  if (half_theta > PT_MAX_HT) return false;
  int best_tch = 0, best_tc = 0;
  double best = 1e30;
  for (int tch = 128; tch <= PT_MAX_THREADS; tch *= 2) {
    const int tc = tch - 2 * half_rho;
    if (tc < 32) continue;
    const double cost = static_cast<double>(tch) / tc + (tch < 256 ? 0.25 : 0.0);
    if (cost < best - 1e-9) {
      best = cost;
      best_tch = tch;
      best_tc = tc;
    }
  }
  if (!best_tch) return false;
  const int cand = ((PT_TR + half_theta) / (half_theta + 1)) *
                   ((best_tc + half_rho) / (half_rho + 1));
  int np2 = 1;
  while (np2 < cand) np2 <<= 1;
  if (np2 < 1) np2 = 1;
  const size_t bytes =
      static_cast<size_t>(((2 * PT_TR + 2 * half_theta) * best_tch * 4 + PT_TR * best_tch * 2 + 15) &
                          ~15) +
      sizeof(u64) * np2;
  if (bytes > 200 * 1024) return false;
  p->tch = best_tch;
  p->tc = best_tc;
  p->tiles_t = (n_theta + PT_TR - 1) / PT_TR;
  p->tiles_r = (n_rho + best_tc - 1) / best_tc;
  p->n_units = p->tiles_t * p->tiles_r;
  *smem = bytes;
  (void)k;
  return true;
}

#ifdef LD_DEBUG
extern "C" int ld_debug_error_line(void) {
  int v = 0;
  cudaMemcpyFromSymbol(&v, g_ld_debug_line, sizeof(int));
  return v;
}
#endif

PeaksLayout peaks_layout(int batch, int n_theta, int n_rho, int k) {
  // per-frame thresholds and resolved flags (each 256-B padded), the
  // diagnostics area (PF_DIAG words per frame, written by experiment builds
  // only), then the per-unit top-k keys: worst case over the dense kernels
  // (tiles/units of >= 16 rows x >= 32 columns, or bands of PK_ROWS rows)
  const size_t tiles = static_cast<size_t>((n_theta + PT_TR - 1) / PT_TR) * ((n_rho + 31) / 32);
  const size_t bands = static_cast<size_t>((n_theta + PK_ROWS - 1) / PK_ROWS);
  const size_t head = (sizeof(uint32_t) * static_cast<size_t>(batch) + 255) / 256 * 256;
  PeaksLayout L;
  L.gtau = 0;
  L.resolved = head;
  L.diag = 2 * head;
  L.keys = L.diag + sizeof(u64) * static_cast<size_t>(batch) * PF_DIAG;
  // + the peak hint computed from the accumulator itself (searches called
  // without one): header, range keys, chunk maxima
  const size_t keys_end = L.keys + static_cast<size_t>(batch) * (tiles > bands ? tiles : bands) * k * sizeof(u64);
  L.self_hdr = (keys_end + 255) / 256 * 256;
  L.self_keys = L.self_hdr + HINT_HDR_BYTES;
  L.self_segmax = L.self_keys + hint_self_keys_bytes(batch, n_theta, n_rho);
  L.total = L.self_segmax +
            sizeof(uint32_t) * static_cast<size_t>(batch) * seg_count(static_cast<int64_t>(n_theta) * n_rho);
  return L;
}

size_t peaks_workspace_bytes(int batch, int n_theta, int n_rho, int k) {
  return peaks_layout(batch, n_theta, n_rho, k).total;
}

static AttrOnce g_tile_attr[PT_MAX_HT + 1];
static AttrOnce g_stream_attr[2][PT_MAX_HT + 1];
static AttrOnce g_warp_attr[4];
static AttrOnce g_fused_attr[5];

// The fused hinted search: 512 threads per CTA; two CTAs per SM (64
// registers) for batches that fill the GPU, else one (128 registers: the
// window tests' loads and chains stay in registers), in clusters of G = 2..8
// CTAs per frame while the frames alone would leave most SMs idle.
template <int NT, int G, int MINB>
static cudaError_t launch_fused_g(const PeaksParams &p, AttrOnce &attr, cudaStream_t stream) {
  auto kern = peaks_fused_kernel<NT, G, MINB>;
  cudaError_t e = ensure_smem_attr(attr, kern, static_cast<int>(PF_SMEM));
  if (e != cudaSuccess) return e;
  return launch_ex(kern, dim3(p.batch * G), dim3(NT), PF_SMEM, stream, G, p);
}

static cudaError_t launch_fused(const PeaksParams &p, int sms, cudaStream_t stream) {
  if (p.batch >= sms) return launch_fused_g<512, 1, 2>(p, g_fused_attr[0], stream);
  const int per = sms / p.batch;
  cudaError_t e = cudaErrorInvalidClusterSize;
  if (per >= 8) e = launch_fused_g<512, 8, 1>(p, g_fused_attr[4], stream);
  else if (per >= 4) e = launch_fused_g<512, 4, 1>(p, g_fused_attr[3], stream);
  else if (per >= 2) e = launch_fused_g<512, 2, 1>(p, g_fused_attr[2], stream);
  if (e != cudaErrorLaunchOutOfResources && e != cudaErrorInvalidClusterSize) return e;
  cudaGetLastError();  // no room for a cluster (or none asked for): one CTA per frame
  return launch_fused_g<512, 1, 1>(p, g_fused_attr[1], stream);
}


cudaError_t launch_peaks(const PeaksParams &p_in, uint32_t flags, cudaStream_t stream) {
  PeaksParams p = p_in;
  size_t smem = 0;
  const bool force_band = (flags & LD_PEAKS_FORCE_BAND) != 0;
  const bool force_tile = (flags & LD_PEAKS_FORCE_TILE) != 0;
  const bool force_stream = (flags & LD_PEAKS_FORCE_STREAM) != 0;
  const bool dense_only = (flags & LD_PEAKS_DENSE) != 0;
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int cpt = 0;
  // candidate rows [cand_t0, cand_t1): the planners chunk those rows only;
  // the tiled kernel has no row restriction and is skipped when one is set
  const int n_cand = p.cand_t1 - p.cand_t0;
  const bool restricted = p.cand_t0 != 0 || p.cand_t1 != p.n_theta || p.theta_offset != 0;
  p.resolved = nullptr;
  if (n_cand <= 0) {  // no candidate rows: the merge writes sentinels and 0 peaks
    p.n_units = 0;
    return launch_ex(peaks_merge_kernel, dim3(p.batch), dim3(PK_THREADS), 0, stream, 1, p);
  }
  const bool dense_cheap = !force_band && !force_tile && !force_stream &&
      peaks_warp_plan(p.batch, n_cand, p.n_rho, p.half_theta, p.half_rho, p.k, sms, &p, &smem);
  const bool dense_stream = !dense_cheap && !force_band && !force_tile &&
      peaks_stream_plan(p.batch, n_cand, p.n_rho, p.half_theta, p.half_rho, p.k, sms, &p, &cpt,
                        &smem);
  if (dense_cheap || dense_stream) {
    // the hint (and with it the sparse search) serves the warp and streaming kernels
    PeaksParams ps = p;
    const int64_t wcells = static_cast<int64_t>(2 * p.half_theta + 1) * (2 * p.half_rho + 1);
    if (!ps.hint_hdr && !dense_only && ps.self_hdr && wcells * p.k <= (1 << 20)) {
      // no hint from voting: take it from the accumulator (one read of it)
      // for the same fused search (R25, R30: the result is unchanged)
      const cudaError_t eh = launch_hint_from_acc(p.acc, p.batch, p.n_theta, p.n_rho, p.cand_t0,
                                                  p.cand_t1, ps.self_hdr, ps.self_keys,
                                                  ps.self_segmax, stream);
      if (eh != cudaSuccess) return eh;
      ps.hint_hdr = p.hint_hdr = ps.self_hdr;
      ps.hint_keys = p.hint_keys = ps.self_keys;
      ps.segmax = p.segmax = ps.self_segmax;
    }
    const bool sparse_ok = ps.hint_hdr && ps.segmax && !dense_only;
    // the bound, the sparse search and its top k in one launch per frame;
    // dense-only searches take the bound alone
    if (ps.hint_hdr && wcells * p.k <= (1 << 20)) {
      ps.resolved = sparse_ok ? p_in.resolved : nullptr;
      if (!sparse_ok) ps.segmax = nullptr;
      const cudaError_t em = launch_fused(ps, sms, stream);
      if (em != cudaSuccess) return em;
      p.resolved = ps.resolved;
    } else {
      p.hint_hdr = nullptr;
      p.hint_keys = nullptr;
      const cudaError_t em = cudaMemsetAsync(p.gtau, 0, sizeof(uint32_t) * p.batch, stream);
      if (em != cudaSuccess) return em;
    }
  }
  if (dense_cheap) {
    WarpKernel kern = warp_kernel(p.half_theta);
    cudaError_t e = ensure_smem_attr(g_warp_attr[p.half_theta], kern, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    dim3 g1((p.n_units + PW_W - 1) / PW_W, p.batch);
    e = launch_ex(kern, g1, dim3(32 * PW_W), smem, stream, 1, p);
    if (e != cudaSuccess) return e;
  } else if (dense_stream) {
    StreamKernel kern = stream_kernel(p.half_theta, cpt);
    cudaError_t e = ensure_smem_attr(g_stream_attr[cpt == 4][p.half_theta], kern, 220 * 1024);
    if (e != cudaSuccess) return e;
    dim3 g1(p.n_units, p.batch);
    e = launch_ex(kern, g1, dim3(p.st_nt), smem, stream, 1, p);
    if (e != cudaSuccess) return e;
  } else if (!force_band && !restricted &&
             peaks_tile_plan(p.n_theta, p.n_rho, p.half_theta, p.half_rho, p.k, &p, &smem)) {
    TileKernel kern = tile_kernel(p.half_theta);
    cudaError_t e = ensure_smem_attr(g_tile_attr[p.half_theta], kern, 200 * 1024);
    if (e != cudaSuccess) return e;
    dim3 g1(p.n_units, p.batch);
    e = launch_ex(kern, g1, dim3(p.tch), smem, stream, 1, p);
    if (e != cudaSuccess) return e;
  } else {
    p.n_units = (n_cand + PK_ROWS - 1) / PK_ROWS;
    dim3 g1(p.n_units, p.batch);
    const cudaError_t e = launch_ex(peaks_band_kernel, g1, dim3(PK_THREADS), 0, stream, 1, p);
    if (e != cudaSuccess) return e;
  }
  return launch_ex(peaks_merge_kernel, dim3(p.batch), dim3(PK_THREADS), 0, stream, 1, p);
}

}  // namespace ld
