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
// Kernel 1 (frames x theta bands of PK_ROWS rows): each thread tests cells of
// the band; a cell whose key is not above the band's running K-th best key is
// skipped before the window scan.  Candidates are buffered in shared memory and
// merged into the band's top-K with a bitonic sort when a chunk produced any.
// Kernel 2 (one CTA per frame): merges the bands' top-K lists.
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
  u64 *out = p.band_keys + (static_cast<int64_t>(f) * p.n_bands + band) * p.k;
  const int ntop = s_ntop;
  for (int i = threadIdx.x; i < p.k; i += PK_THREADS) out[i] = i < ntop ? top[i] : 0ull;
}

__global__ void __launch_bounds__(PK_THREADS) peaks_merge_kernel(const PeaksParams p) {
  __shared__ u64 buf[PK_BUF];
  __shared__ u64 top[LD_MAX_K];
  __shared__ int s_ntop;
  const int f = blockIdx.x;
  const u64 *in = p.band_keys + static_cast<int64_t>(f) * p.n_bands * p.k;
  const int n_in = p.n_bands * p.k;
  if (threadIdx.x == 0) s_ntop = 0;
  __syncthreads();
  for (int base = 0; base < n_in; base += PK_CHUNK) {
    const int nb = min(PK_CHUNK, n_in - base);
    for (int i = threadIdx.x; i < nb; i += PK_THREADS) buf[i] = in[base + i];
    __syncthreads();
    merge_topk(buf, nb, top, &s_ntop, p.k);
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

size_t peaks_workspace_bytes(int batch, int n_theta, int k) {
  const int nb = (n_theta + PK_ROWS - 1) / PK_ROWS;
  return static_cast<size_t>(batch) * nb * k * sizeof(u64);
}

cudaError_t launch_peaks(const PeaksParams &p, cudaStream_t stream) {
  dim3 g1(p.n_bands, p.batch);
  peaks_band_kernel<<<g1, PK_THREADS, 0, stream>>>(p);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  peaks_merge_kernel<<<p.batch, PK_THREADS, 0, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ld
