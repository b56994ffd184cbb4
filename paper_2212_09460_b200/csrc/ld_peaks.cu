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
// Kernel 1, fast path (peaks_tile_kernel): separable window maximum over
// 16 x tc tiles, see below.  Kernel 1, generic fallback for very large windows
// (peaks_band_kernel: frames x theta bands of PK_ROWS rows): each thread tests
// cells of the band by a window scan with early exit; a cell whose key is not
// above the band's running K-th best key is skipped first.  Candidates are
// buffered in shared memory and merged into the band's top-K with a bitonic
// sort.  Kernel 2 (one CTA per frame): merges the per-unit top-K lists.
#include <cstdlib>

#include "ld_internal.cuh"

namespace ld {

typedef unsigned long long u64;

constexpr int PK_CHUNK = 2 * PK_THREADS;        // cells tested per round
constexpr int PK_BUF = PK_CHUNK + LD_MAX_K;     // candidate buffer (power of 2)
static_assert((PK_BUF & (PK_BUF - 1)) == 0, "PK_BUF must be a power of two");

__device__ __forceinline__ u64 mk_key(uint32_t v, uint32_t idx) {
  return (static_cast<u64>(v) << 32) | static_cast<u64>(0xFFFFFFFFu - idx);
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
  __shared__ u64 buf[PK_BUF];
  __shared__ u64 top[LD_MAX_K];
  __shared__ int s_nbuf, s_ntop;

  const int band = blockIdx.x, f = blockIdx.y;
  const int t0 = band * PK_ROWS;
  const int nr = min(PK_ROWS, p.n_theta - t0);
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
          const u64 key = mk_key(v, static_cast<uint32_t>(t * p.n_rho + r));
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

__global__ void __launch_bounds__(PK_THREADS) peaks_merge_kernel(const PeaksParams p) {
  __shared__ u64 buf[PK_BUF];
  __shared__ u64 top[LD_MAX_K];
  __shared__ int s_ntop;
  const int f = blockIdx.x;
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
bool peaks_tile_plan(int n_theta, int n_rho, int half_theta, int half_rho, int k, PeaksParams *p,
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

size_t peaks_workspace_bytes(int batch, int n_theta, int n_rho, int k) {
  // worst case over both kernels: tiles with tc >= 32, or bands of PK_ROWS rows
  const size_t tiles = static_cast<size_t>((n_theta + PT_TR - 1) / PT_TR) * ((n_rho + 31) / 32);
  const size_t bands = static_cast<size_t>((n_theta + PK_ROWS - 1) / PK_ROWS);
  return static_cast<size_t>(batch) * (tiles > bands ? tiles : bands) * k * sizeof(u64);
}

static bool g_tile_attr[64][PT_MAX_HT + 1];

cudaError_t launch_peaks(const PeaksParams &p_in, cudaStream_t stream) {
  PeaksParams p = p_in;
  size_t smem = 0;
  const char *env = getenv("LD_PEAKS_KERNEL");
  const bool force_band = env && env[0] == 'b';
  if (!force_band && peaks_tile_plan(p.n_theta, p.n_rho, p.half_theta, p.half_rho, p.k, &p, &smem)) {
    TileKernel kern = tile_kernel(p.half_theta);
    int dev = 0;
    cudaGetDevice(&dev);
    if (!g_tile_attr[dev & 63][p.half_theta]) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           200 * 1024);
      if (e != cudaSuccess) return e;
      g_tile_attr[dev & 63][p.half_theta] = true;
    }
    dim3 g1(p.n_units, p.batch);
    kern<<<g1, p.tch, smem, stream>>>(p);
  } else {
    p.n_units = (p.n_theta + PK_ROWS - 1) / PK_ROWS;
    dim3 g1(p.n_units, p.batch);
    peaks_band_kernel<<<g1, PK_THREADS, 0, stream>>>(p);
  }
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  peaks_merge_kernel<<<p.batch, PK_THREADS, 0, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ld
