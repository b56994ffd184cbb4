// ld_lanes.cu -- NEXT 3: SPEC's lanes module on the GPU,
// completing Fig. 1 step 4 ("draw the lane lines"; P:185 MATLAB
// houghpeaks, Fig. 12 houghlines).  DESIGN R26-R28, section 6.6.
//
//  * greedy non-maximum suppression (SPEC find_peaks): k rounds of
//    a grid-wide arg-max over the eligible, unsuppressed cells of every frame
//    (64-bit key (votes << 32) | ~index, one atomicMax per CTA) followed by a
//    per-frame pick kernel that appends the winner and marks its window in a
//    suppression bitmap.  Exact for every input; each round streams the
//    accumulators once (this is not the benchmarked path);
//  * peak_to_line: one thread per peak, double precision with
//    every product, quotient and sum rounded on its own (__dmul_rn, __ddiv_rn,
//    __dadd_rn: no contraction), the oracle's exact operation sequence;
//  * extract_segments: one warp per peak walks the rasterised line
//    32 samples at a time (ballot of the white samples) and applies the gap
//    rule in walk order.
#include "ld_internal.cuh"

namespace ld {

typedef unsigned long long u64;

// ---------------------------------------------------------------------------
// greedy NMS
// ---------------------------------------------------------------------------
constexpr int NMS_THREADS = 512;
constexpr int NMS_CELLS_PER_CTA = NMS_THREADS * 8;

__global__ void __launch_bounds__(NMS_THREADS) nms_argmax_kernel(const NmsParams p) {
  __shared__ u64 red[NMS_THREADS / 32];
  const int f = blockIdx.y;
  NmsState &st = p.state[f];
  if (st.done) return;
  const uint32_t thr = max(st.thr, p.floor_votes);
  const int64_t cells = static_cast<int64_t>(p.n_theta) * p.n_rho;
  const uint32_t *A = p.acc + static_cast<int64_t>(f) * cells;
  const uint32_t *bits = p.bitmap + static_cast<int64_t>(f) * p.bitmap_words;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * NMS_CELLS_PER_CTA;
  u64 best = 0ull;
  for (int64_t i = c0 + threadIdx.x; i < min(c0 + NMS_CELLS_PER_CTA, cells); i += NMS_THREADS) {
    const uint32_t v = __ldg(A + i);
    if (v < thr) continue;
    if ((bits[i >> 5] >> (i & 31)) & 1u) continue;
    const u64 key = (static_cast<u64>(v) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(i));
    best = key > best ? key : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const u64 other = __shfl_xor_sync(0xffffffffu, best, o);
    best = other > best ? other : best;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    best = threadIdx.x < NMS_THREADS / 32 ? red[threadIdx.x] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const u64 other = __shfl_xor_sync(0xffffffffu, best, o);
      best = other > best ? other : best;
    }
    if (threadIdx.x == 0 && best) atomicMax(&st.best, best);
  }
}

__global__ void __launch_bounds__(256) nms_pick_kernel(const NmsParams p) {
  const int f = blockIdx.x;
  NmsState &st = p.state[f];
  __shared__ int s_pick;
  __shared__ int s_t, s_r;
  if (threadIdx.x == 0) {
    s_pick = 0;
    const u64 key = st.best;
    if (!st.done) {
      if (key == 0ull) {
        st.done = 1u;
      } else {
        const uint32_t v = static_cast<uint32_t>(key >> 32);
        const uint32_t idx = 0xFFFFFFFFu - static_cast<uint32_t>(key);
        if (st.npicks == 0) {
          // the first pick is the global maximum gmax (it is >= the floor);
          // eligible from now on: v * den >= num * gmax, i.e. v >= thr
          const u64 num = static_cast<u64>(p.ratio_num) * v;
          const u64 thr = (num + p.ratio_den - 1) / p.ratio_den;
          const u64 floor_v = p.floor_votes;
          const u64 t = thr > floor_v ? thr : floor_v;
          st.thr = t > 0xFFFFFFFFull ? 0xFFFFFFFFu : static_cast<uint32_t>(t);
          if (t > v) st.done = 1u;  // a ratio above 1: not even the maximum qualifies
        }
        if (!st.done) {
          const int t = static_cast<int>(idx / static_cast<uint32_t>(p.n_rho));
          const int r = static_cast<int>(idx - static_cast<uint32_t>(t) * p.n_rho);
          ld_peak *out = p.peaks + static_cast<int64_t>(f) * p.k + st.npicks;
          out->theta_bin = t;
          out->rho_bin = r;
          out->votes = v;
          st.npicks += 1;
          if (static_cast<int>(st.npicks) >= p.k) st.done = 1u;
          s_pick = 1;
          s_t = t;
          s_r = r;
        }
        st.best = 0ull;
      }
    }
  }
  __syncthreads();
  if (!s_pick) return;
  // suppress the clipped window of the pick (itself included)
  uint32_t *bits = p.bitmap + static_cast<int64_t>(f) * p.bitmap_words;
  const int ta = max(s_t - p.half_theta, 0), tb = min(s_t + p.half_theta, p.n_theta - 1);
  const int ra = max(s_r - p.half_rho, 0), rb = min(s_r + p.half_rho, p.n_rho - 1);
  const int wc = rb - ra + 1;
  const int cells = (tb - ta + 1) * wc;
  for (int c = threadIdx.x; c < cells; c += blockDim.x) {
    const int64_t i = static_cast<int64_t>(ta + c / wc) * p.n_rho + (ra + c % wc);
    atomicOr(bits + (i >> 5), 1u << (i & 31));
  }
}

__global__ void nms_finish_kernel(const NmsParams p) {
  const int f = blockIdx.x;
  const int n = static_cast<int>(p.state[f].npicks);
  for (int i = n + threadIdx.x; i < p.k; i += blockDim.x) {
    ld_peak *out = p.peaks + static_cast<int64_t>(f) * p.k + i;
    out->theta_bin = -1;
    out->rho_bin = -1;
    out->votes = 0u;
  }
  if (threadIdx.x == 0) p.n_peaks[f] = n;
}

cudaError_t launch_nms(const NmsParams &p, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(p.state, 0, sizeof(NmsState) * p.batch, stream);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(p.bitmap, 0, sizeof(uint32_t) * static_cast<size_t>(p.bitmap_words) * p.batch,
                      stream);
  if (e != cudaSuccess) return e;
  const int64_t cells = static_cast<int64_t>(p.n_theta) * p.n_rho;
  dim3 g1(static_cast<unsigned>((cells + NMS_CELLS_PER_CTA - 1) / NMS_CELLS_PER_CTA), p.batch);
  for (int i = 0; i < p.k; ++i) {
    nms_argmax_kernel<<<g1, NMS_THREADS, 0, stream>>>(p);
    nms_pick_kernel<<<p.batch, 256, 0, stream>>>(p);
    note_launch(2);
  }
  nms_finish_kernel<<<p.batch, 256, 0, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// peak_to_line and extract_segments
// ---------------------------------------------------------------------------
__device__ __forceinline__ int32_t round_half_up(double v) {
  return static_cast<int32_t>(floor(__dadd_rn(v, 0.5)));
}

__global__ void peak_lines_kernel(const LanesParams p, const __grid_constant__ TrigTable trig) {
  const int f = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.k) return;
  ld_segment *out = p.lines + static_cast<int64_t>(f) * p.k + i;
  int32_t *hit = p.hit + static_cast<int64_t>(f) * p.k + i;
  *hit = 0;
  if (i >= p.n_peaks[f]) return;
  const ld_peak pk = p.peaks[static_cast<int64_t>(f) * p.k + i];
  if (pk.theta_bin < 0 || pk.theta_bin >= p.n_theta) return;
  const double c = __ddiv_rn(static_cast<double>(trig.c[pk.theta_bin]), 32768.0);
  const double s = __ddiv_rn(static_cast<double>(trig.s[pk.theta_bin]), 32768.0);
  const double rho = static_cast<double>(pk.rho_bin - p.rho_offset);
  const double W1 = static_cast<double>(p.width - 1), H1 = static_cast<double>(p.height - 1);
  double px[4], py[4];
  int n = 0;
  const double xs[2] = {0.0, W1}, ys[2] = {0.0, H1};
  if (s != 0.0) {
    for (int j = 0; j < 2; ++j) {
      const double y = __ddiv_rn(__dsub_rn(rho, __dmul_rn(xs[j], c)), s);
      if (y >= 0.0 && y <= H1) {
        px[n] = xs[j];
        py[n] = y;
        ++n;
      }
    }
  }
  if (c != 0.0) {
    for (int j = 0; j < 2; ++j) {
      const double x = __ddiv_rn(__dsub_rn(rho, __dmul_rn(ys[j], s)), c);
      if (x >= 0.0 && x <= W1) {
        px[n] = x;
        py[n] = ys[j];
        ++n;
      }
    }
  }
  if (n == 0) return;
  int lo = 0, hi = 0;
  double plo = __dadd_rn(__dmul_rn(-px[0], s), __dmul_rn(py[0], c)), phi = plo;
  for (int j = 1; j < n; ++j) {
    const double q = __dadd_rn(__dmul_rn(-px[j], s), __dmul_rn(py[j], c));
    if (q < plo) {
      plo = q;
      lo = j;
    }
    if (q > phi) {
      phi = q;
      hi = j;
    }
  }
  int32_t ax = round_half_up(px[lo]), ay = round_half_up(py[lo]);
  int32_t bx = round_half_up(px[hi]), by = round_half_up(py[hi]);
  if (bx < ax || (bx == ax && by < ay)) {
    const int32_t tx = ax, ty = ay;
    ax = bx;
    ay = by;
    bx = tx;
    by = ty;
  }
  out->x0 = ax;
  out->y0 = ay;
  out->x1 = bx;
  out->y1 = by;
  *hit = 1;
}

// one warp per (frame, peak slot)
__global__ void extract_segments_kernel(const LanesParams p, const __grid_constant__ TrigTable trig) {
  const int f = blockIdx.y;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= p.k) return;  // whole warp
  int32_t *nseg = p.n_segs + static_cast<int64_t>(f) * p.k + i;
  ld_segment *segs = p.segs + (static_cast<int64_t>(f) * p.k + i) * p.max_segs;
  if (i >= p.n_peaks[f]) {
    if (lane == 0) *nseg = 0;
    return;
  }
  const ld_peak pk = p.peaks[static_cast<int64_t>(f) * p.k + i];
  // a peak from another table size (or a sentinel inside n_peaks) has no line
  // here: no segments, and no read outside the table
  if (pk.theta_bin < 0 || pk.theta_bin >= p.n_theta) {
    if (lane == 0) *nseg = 0;
    return;
  }
  const int32_t ci = trig.c[pk.theta_bin], si = trig.s[pk.theta_bin];
  if (ci == 0 && si == 0) {
    if (lane == 0) *nseg = 0;
    return;
  }
  const double c = __ddiv_rn(static_cast<double>(ci), 32768.0);
  const double s = __ddiv_rn(static_cast<double>(si), 32768.0);
  const double rho = static_cast<double>(pk.rho_bin - p.rho_offset);
  const bool along_x = (si < 0 ? -si : si) >= (ci < 0 ? -ci : ci);
  const int n = along_x ? p.width : p.height;
  const uint8_t *bin = p.binary + static_cast<int64_t>(f) * p.bin_frame_stride;
  int count = 0;
  int run_a = -1, run_b = -1, ax = 0, ay = 0, bx = 0, by = 0;  // warp-uniform
  for (int base = 0; base < n; base += 32) {
    const int idx = base + lane;
    int x = 0, y = 0;
    bool white = false;
    if (idx < n) {
      if (along_x) {
        x = idx;
        y = round_half_up(__ddiv_rn(__dsub_rn(rho, __dmul_rn(static_cast<double>(idx), c)), s));
      } else {
        y = idx;
        x = round_half_up(__ddiv_rn(__dsub_rn(rho, __dmul_rn(static_cast<double>(idx), s)), c));
      }
      white = x >= 0 && x < p.width && y >= 0 && y < p.height &&
              bin[static_cast<int64_t>(y) * p.bin_pitch + x] == 255;
    }
    uint32_t m = __ballot_sync(0xffffffffu, white);
    while (m) {  // the white samples of this step, in walk order (uniform)
      const int b = __ffs(m) - 1;
      m &= m - 1u;
      const int wi = base + b;
      const int wx = __shfl_sync(0xffffffffu, x, b), wy = __shfl_sync(0xffffffffu, y, b);
      if (run_a >= 0 && wi - run_b - 1 > p.fill_gap) {
        const int64_t dx = bx - ax, dy = by - ay;
        if (dx * dx + dy * dy >= static_cast<int64_t>(p.min_len) * p.min_len) {
          if (lane == 0 && count < p.max_segs) segs[count] = ld_segment{ax, ay, bx, by};
          ++count;
        }
        run_a = -1;
      }
      if (run_a < 0) {
        run_a = wi;
        ax = wx;
        ay = wy;
      }
      run_b = wi;
      bx = wx;
      by = wy;
    }
  }
  if (run_a >= 0) {
    const int64_t dx = bx - ax, dy = by - ay;
    if (dx * dx + dy * dy >= static_cast<int64_t>(p.min_len) * p.min_len) {
      if (lane == 0 && count < p.max_segs) segs[count] = ld_segment{ax, ay, bx, by};
      ++count;
    }
  }
  if (lane == 0) *nseg = count;
}

cudaError_t launch_peak_lines(const LanesParams &p, const TrigTable &trig, cudaStream_t stream) {
  dim3 g((p.k + 127) / 128, p.batch);
  peak_lines_kernel<<<g, 128, 0, stream>>>(p, trig);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_extract_segments(const LanesParams &p, const TrigTable &trig,
                                    cudaStream_t stream) {
  dim3 g((p.k + 7) / 8, p.batch);
  extract_segments_kernel<<<g, 256, 0, stream>>>(p, trig);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ld
