// Streaming-read probe for the peaks kernels' access pattern: a [B][nt][nr]
// uint32 array read (a) by plain grid-stride uint4 loads, (b) per warp as
// 256-column strips x row chunks with lane-strided 4-byte loads PF rows ahead
// (registers), (c) the same strips through a per-warp shared-memory ring fed
// by 1040-byte cp.async.bulk copies.  Prints GB/s.  Not part of libld.so.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe tools/stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void plain(const uint4 *a, size_t n4, uint32_t *sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(a + i);
    acc = max(acc, max(max(v.x, v.y), max(v.z, v.w)));
  }
  if (acc == 0xFFFFFFFFu) sink[0] = acc;
}

struct Geo { int nt, nr, sw, strips, tb, chunks, batch; };

template <int PF>
__global__ void __launch_bounds__(256, 2) strips_ldg(const uint32_t *acc, Geo g, uint32_t *sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x * 8 + warp, f = blockIdx.y;
  if (unit >= g.strips * g.chunks) return;
  const int strip = unit / g.chunks, chunk = unit % g.chunks;
  const int cbase = max(strip * g.sw - 29, 0);
  const int t0 = chunk * g.tb, t1 = min(t0 + g.tb, g.nt);
  const uint32_t *fr = acc + (size_t)f * g.nt * g.nr;
  uint32_t m = 0;
  uint32_t buf[PF][8];
  int r = t0;
  for (int k = 0; k < PF; ++k, ++r)
    for (int q = 0; q < 8; ++q) buf[k][q] = (r < t1 && cbase + lane + 32 * q < g.nr) ? __ldg(fr + (size_t)r * g.nr + cbase + lane + 32 * q) : 0u;
  for (int t = t0; t < t1; t += PF) {
#pragma unroll
    for (int k = 0; k < PF; ++k) {
#pragma unroll
      for (int q = 0; q < 8; ++q) m = max(m, buf[k][q]);
      const int rr = t + PF + k;
#pragma unroll
      for (int q = 0; q < 8; ++q) buf[k][q] = (rr < t1 && cbase + lane + 32 * q < g.nr) ? __ldg(fr + (size_t)rr * g.nr + cbase + lane + 32 * q) : 0u;
    }
  }
  if (__any_sync(0xffffffffu, m == 0xFFFFFFFFu)) sink[0] = m;
}

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int RING, bool HINT>
__global__ void __launch_bounds__(256, 2) strips_bulk(const uint32_t *acc, Geo g, uint32_t *sink) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *ring = reinterpret_cast<uint32_t *>(sm) + warp * RING * 260;
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 8 * RING * 260 * 4) + warp * RING;
  const int unit = blockIdx.x * 8 + warp, f = blockIdx.y;
  if (unit >= g.strips * g.chunks) return;
  const int strip = unit / g.chunks, chunk = unit % g.chunks;
  const int cbase = max(strip * g.sw - 29, 4);
  const int t0 = chunk * g.tb, t1 = min(t0 + g.tb, g.nt);
  const uint32_t *fr = acc + (size_t)f * g.nt * g.nr;
  if (lane == 0) {
    for (int i = 0; i < RING; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + i)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int r) {
    const int slot = (r - t0) % RING;
    if (lane == 0) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(fr + (size_t)r * g.nr + cbase) & ~(uintptr_t)15;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + slot)), "r"(1040u) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(ring + slot * 260)),
                   "l"(a), "r"(1040u), "r"(su32(bar + slot)) : "memory");
    }
  };
  int ni = t0;
  for (; ni < min(t0 + RING, t1); ++ni) issue(ni);
  uint32_t m = 0;
  for (int r = t0; r < t1; ++r) {
    const int slot = (r - t0) % RING;
    const uint32_t par = ((r - t0) / RING) & 1;
    if (HINT)
      asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 0x989680;\n\t@!p bra W_%=;\n}" ::"r"(su32(bar + slot)), "r"(par) : "memory");
    else
      asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su32(bar + slot)), "r"(par) : "memory");
#pragma unroll
    for (int q = 0; q < 8; ++q) m = max(m, ring[slot * 260 + lane + 32 * q]);
    __syncwarp();
    if (ni < t1) issue(ni++);
  }
  if (__any_sync(0xffffffffu, m == 0xFFFFFFFFu)) sink[0] = m;
}


// the warp-strip peaks kernel's skeleton: register ring of 2 HT + (1 + PF) G
// rows unrolled over one ring period, a per-group quick reject (ballot), and
// optionally the per-frame threshold read (relaxed, consumed one group later)
template <int HT, int PF, bool GTAU>
__global__ void __launch_bounds__(256, 2) strips_ring(const uint32_t *acc, Geo g, uint32_t *gtau, uint32_t *sink) {
  constexpr int G = 2, NV = G + 2 * HT, R = NV + PF * G, U = R / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x * 8 + warp, f = blockIdx.y;
  if (unit >= g.strips * g.chunks) return;
  const int strip = unit / g.chunks, chunk = unit % g.chunks;
  const int cbase = max(strip * g.sw - 29, 0);
  const int t0 = chunk * g.tb, t1 = min(t0 + g.tb, g.nt);
  const bool all_in = cbase + 256 <= g.nr;
  const uint32_t *rowp = acc + (size_t)f * g.nt * g.nr + (size_t)(t0 - HT) * g.nr + cbase + lane;
  int rnext = t0 - HT;
  auto load_row = [&](uint32_t (&d)[8]) {
    if (rnext >= 0 && rnext < g.nt) {
      if (all_in) {
#pragma unroll
        for (int q = 0; q < 8; ++q) d[q] = __ldg(rowp + 32 * q);
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) d[q] = (cbase + lane + 32 * q < g.nr) ? __ldg(rowp + 32 * q) : 0u;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) d[q] = 0u;
    }
    rowp += g.nr;
    ++rnext;
  };
  uint32_t ring[R][8];
#pragma unroll
  for (int k = 0; k < NV + (PF - 1) * G; ++k) load_row(ring[k]);
  uint32_t tau = 0xF0000000u, gt_next = 0, hits = 0;
  for (int gp = t0; gp < t1; gp += U * G) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int g0 = gp + u * G;
      if (g0 >= t1) break;
      if (g0 + PF * G < t1) {
#pragma unroll
        for (int k = 0; k < G; ++k) load_row(ring[(u * G + NV + (PF - 1) * G + k) % R]);
      }
      if (GTAU) {
        uint32_t gt = gt_next;
        if (lane == 0) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gt_next) : "l"(gtau + f) : "memory");
        tau = max(tau, __shfl_sync(0xffffffffu, gt, 0));
      }
      uint32_t hm = 0;
#pragma unroll
      for (int i = 0; i < G; ++i)
#pragma unroll
        for (int q = 0; q < 8; ++q) hm = max(hm, ring[(u * G + i + HT) % R][q]);
      if (__any_sync(0xffffffffu, hm >= tau)) ++hits;
    }
  }
  if (hits == 12345) sink[0] = hits;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int i = 0; i < 5; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  Geo g{180, 2939, 198, 15, 56, 4, 256};
  const size_t n = (size_t)g.batch * g.nt * g.nr;
  uint32_t *acc, *sink;
  cudaMalloc(&acc, n * 4 + 64);
  cudaMalloc(&sink, 64);
  cudaMemset(acc, 1, n * 4);
  const double gb = n * 4 / 1e9;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float t = timeit([&] { plain<<<sms * 8, 256>>>(reinterpret_cast<const uint4 *>(acc), n / 4, sink); });
  printf("plain uint4           %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  const int units = g.strips * g.chunks;
  dim3 grid((units + 7) / 8, g.batch);
  t = timeit([&] { strips_ldg<1><<<grid, 256>>>(acc, g, sink); });
  printf("strips ldg PF1        %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  t = timeit([&] { strips_ldg<2><<<grid, 256>>>(acc, g, sink); });
  printf("strips ldg PF2        %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  t = timeit([&] { strips_ldg<4><<<grid, 256>>>(acc, g, sink); });
  printf("strips ldg PF4        %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  {
    const int smem = 8 * 10 * 1040 + 8 * 10 * 8;
    cudaFuncSetAttribute(strips_bulk<10, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(strips_bulk<10, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    t = timeit([&] { strips_bulk<10, true><<<grid, 256, smem>>>(acc, g, sink); });
    printf("strips bulk R10 hint  %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
    t = timeit([&] { strips_bulk<10, false><<<grid, 256, smem>>>(acc, g, sink); });
    printf("strips bulk R10 spin  %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  }
  {
    const int smem = 8 * 20 * 1040 + 8 * 20 * 8;
    cudaFuncSetAttribute(strips_bulk<20, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    t = timeit([&] { strips_bulk<20, false><<<grid, 256, smem>>>(acc, g, sink); });
    printf("strips bulk R20 spin  %.3f ms  %.0f GB/s (1 CTA/SM)\n", t, gb / t * 1e3);
  }
  {
    const int smem = 8 * 5 * 1040 + 8 * 5 * 8;
    cudaFuncSetAttribute(strips_bulk<5, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    t = timeit([&] { strips_bulk<5, false><<<grid, 256, smem>>>(acc, g, sink); });
    printf("strips bulk R5 spin   %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  }
  {
    uint32_t *gt;
    cudaMalloc(&gt, 4096);
    cudaMemset(gt, 0, 4096);
    t = timeit([&] { strips_ring<2, 1, false><<<grid, 256>>>(acc, g, gt, sink); });
    printf("ring HT2 PF1          %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
    t = timeit([&] { strips_ring<2, 1, true><<<grid, 256>>>(acc, g, gt, sink); });
    printf("ring HT2 PF1 gtau     %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
    t = timeit([&] { strips_ring<2, 2, false><<<grid, 256>>>(acc, g, gt, sink); });
    printf("ring HT2 PF2          %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
    t = timeit([&] { strips_ring<2, 2, true><<<grid, 256>>>(acc, g, gt, sink); });
    printf("ring HT2 PF2 gtau     %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
    t = timeit([&] { strips_ring<2, 3, true><<<grid, 256>>>(acc, g, gt, sink); });
    printf("ring HT2 PF3 gtau     %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
