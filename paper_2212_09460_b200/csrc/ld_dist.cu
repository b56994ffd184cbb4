// ld_dist.cu -- device-side pieces of the theta-sharded multi-GPU path
// (DESIGN section 8): the exchange of band edge sets as
// fixed-size bitmaps (so the all_gather needs no host-known sizes) and the
// merge of per-rank top-k lists.  Paper: the theta partitioning of the voting
// lifted across GPUs; peaks P:100 with the deterministic key of
// DESIGN R14.
//
//  * edges_to_bitmask_kernel: one bit per owned pixel, set for each listed
//    edge (atomicOr: list order is unspecified, R15).
//  * bitmask_to_edges_kernel: the set back to a list.  A warp takes a block
//    of 16 columns x 32 rows (lane l: row l's 16-bit field) and emits it in
//    lane order, so 32 consecutive list entries cover a ~16 x 20-pixel region
//    (the voting kernel's bank-conflict-free window, ld_hough.cu); one list
//    reservation (atomicAdd) per warp.
//  * merge_peak_lists_kernel: the top k of several top-k lists by the key
//    (votes, -theta, -rho) -- one CTA, bitonic sort in shared memory.
#include "ld_internal.cuh"

namespace ld {

__global__ void __launch_bounds__(256) edges_to_bitmask_kernel(const uint32_t *edges,
                                                              const uint32_t *count, int words,
                                                              int row_begin, int rows,
                                                              uint32_t *bits) {
  const uint32_t n = *count;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t e = edges[i];
    const int x = static_cast<int>(e & 0xFFFFu), y = static_cast<int>(e >> 16) - row_begin;
    if (y >= 0 && y < rows)
      atomicOr(bits + static_cast<int64_t>(y) * words + (x >> 5), 1u << (x & 31));
  }
}

struct BlockTable {
  int32_t row_begin[LD_MAX_BLOCKS];
  int32_t rows[LD_MAX_BLOCKS];
};

// grid: (ceil(words*2 / 4) warp-columns of 16 px, ceil(rows_max / 32), n_blocks); 4 warps per CTA
__global__ void __launch_bounds__(128) bitmask_to_edges_kernel(const uint32_t *bits, int width,
                                                               int words, int block_stride_rows,
                                                               const __grid_constant__ BlockTable tb,
                                                               uint32_t *edges, int64_t capacity,
                                                               uint32_t *count) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col16 = blockIdx.x * 4 + warp;  // 16-pixel column field
  const int blk = blockIdx.z;
  const int r = blockIdx.y * 32 + lane;     // row inside the block
  const int nrows = tb.rows[blk];
  if (col16 * 16 >= width) return;          // whole warp
  uint32_t m = 0u;
  if (r < nrows) {
    const uint32_t w = bits[(static_cast<int64_t>(blk) * block_stride_rows + r) * words + (col16 >> 1)];
    m = (col16 & 1) ? (w >> 16) : (w & 0xFFFFu);
  }
  const uint32_t c = __popc(m);
  uint32_t incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  if (total == 0) return;
  uint32_t base = 0;
  if (lane == 0) base = atomicAdd(count, total);
  base = __shfl_sync(0xffffffffu, base, 0);
  uint32_t pos = base + incl - c;
  const uint32_t v0 = (static_cast<uint32_t>(tb.row_begin[blk] + r) << 16) |
                      static_cast<uint32_t>(col16 * 16);
  while (m) {
    const int b = __ffs(m) - 1;
    m &= m - 1;
    if (pos < capacity) edges[pos] = v0 + b;
    ++pos;
  }
}

__global__ void __launch_bounds__(256) merge_peak_lists_kernel(const ld_peak *peaks,
                                                              const int32_t *n_peaks, int n_lists,
                                                              int k, int n_rho, ld_peak *out,
                                                              int32_t *n_out) {
  extern __shared__ unsigned long long keys[];
  const int total = n_lists * k;
  int n2 = 1;
  while (n2 < total) n2 <<= 1;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    unsigned long long key = 0ull;
    if (i < total) {
      const int l = i / k, j = i - l * k;
      if (j < n_peaks[l]) {
        const ld_peak p = peaks[i];
        const uint32_t idx = static_cast<uint32_t>(p.theta_bin) * static_cast<uint32_t>(n_rho) +
                             static_cast<uint32_t>(p.rho_bin);
        key = (static_cast<unsigned long long>(p.votes) << 32) | (0xFFFFFFFFu - idx);
      }
    }
    keys[i] = key;
  }
  __syncthreads();
  for (int kk = 2; kk <= n2; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long x = keys[i], y = keys[ixj];
          const bool desc = (i & kk) == 0;
          if (desc ? (x < y) : (x > y)) {
            keys[i] = y;
            keys[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  __shared__ int s_n;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const unsigned long long key = i < total ? keys[i] : 0ull;
    ld_peak p;
    if (key >= (1ull << 32)) {  // a real peak has votes >= 1
      const uint32_t idx = 0xFFFFFFFFu - static_cast<uint32_t>(key);
      p.theta_bin = static_cast<int32_t>(idx / static_cast<uint32_t>(n_rho));
      p.rho_bin = static_cast<int32_t>(idx % static_cast<uint32_t>(n_rho));
      p.votes = static_cast<uint32_t>(key >> 32);
      atomicAdd(&s_n, 1);
    } else {
      p.theta_bin = -1;
      p.rho_bin = -1;
      p.votes = 0u;
    }
    out[i] = p;
  }
  __syncthreads();
  if (threadIdx.x == 0) *n_out = s_n;
}

cudaError_t launch_edges_to_bitmask(const uint32_t *edges, const uint32_t *count, int width,
                                    int row_begin, int rows, uint32_t *bits, int sm_count,
                                    cudaStream_t stream) {
  const int words = (width + 31) / 32;
  cudaError_t e = cudaMemsetAsync(bits, 0, sizeof(uint32_t) * static_cast<size_t>(words) * rows, stream);
  if (e != cudaSuccess) return e;
  edges_to_bitmask_kernel<<<sm_count * 4, 256, 0, stream>>>(edges, count, words, row_begin, rows,
                                                           bits);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_bitmask_to_edges(const uint32_t *bits, int width, int n_blocks,
                                    const int32_t *row_begin, const int32_t *rows,
                                    int block_stride_rows, uint32_t *edges, int64_t capacity,
                                    uint32_t *count, cudaStream_t stream) {
  BlockTable tb;
  int max_rows = 1;
  for (int i = 0; i < LD_MAX_BLOCKS; ++i) {
    tb.row_begin[i] = i < n_blocks ? row_begin[i] : 0;
    tb.rows[i] = i < n_blocks ? rows[i] : 0;
    if (i < n_blocks && rows[i] > max_rows) max_rows = rows[i];
  }
  const int words = (width + 31) / 32;
  cudaError_t e = cudaMemsetAsync(count, 0, sizeof(uint32_t), stream);
  if (e != cudaSuccess) return e;
  const int fields = (width + 15) / 16;
  dim3 grid((fields + 3) / 4, (max_rows + 31) / 32, n_blocks);
  bitmask_to_edges_kernel<<<grid, 128, 0, stream>>>(bits, width, words, block_stride_rows, tb,
                                                    edges, capacity, count);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_merge_peak_lists(const ld_peak *peaks, const int32_t *n_peaks, int n_lists,
                                    int k, int n_rho, ld_peak *out, int32_t *n_out,
                                    cudaStream_t stream) {
  int n2 = 1;
  while (n2 < n_lists * k) n2 <<= 1;
  const size_t smem = sizeof(unsigned long long) * static_cast<size_t>(n2);
  static AttrOnce attr;
  cudaError_t e = ensure_smem_attr(attr, merge_peak_lists_kernel, 200 * 1024);
  if (e != cudaSuccess) return e;
  merge_peak_lists_kernel<<<1, 256, smem, stream>>>(peaks, n_peaks, n_lists, k, n_rho, out, n_out);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ld
