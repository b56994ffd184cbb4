// Voting inner-loop probe (not part of libld.so): warp-ATOMS per clock per SM
// of two address computations for the half-angle paired vote, on synthetic
// conflict-free data (each warp's 32 edges sit on one image row, so every
// theta puts them into <= 32 consecutive bins):
//   0 shift : q = y*S + K; v = x*(+-C) + q; a = (v >> 13) & ~3          (9 / pair)
//   1 wide  : Q = (4y)*(S<<15) + (K<<17) (64-bit); U = (4x)*(+-C<<15) + Q;
//             a = hi32(U) << 2  (hi32(U) = floor(V / 2^15))             (7 / pair)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o vote_probe tools/vote_probe.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

constexpr int EPL = 16, NP = 8, NT = 512;

__device__ __forceinline__ void red_add(uint32_t a) {
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a) : "memory");
}

struct Tab { int c[NP], s[NP]; };

__device__ __forceinline__ uint32_t wide_hi(uint32_t a, int32_t b, unsigned long long c) {
  uint32_t hi;
  asm("{\n\t.reg .b64 u;\n\t.reg .b32 lo;\n\t"
      "mad.wide.s32 u, %1, %2, %3;\n\tmov.b64 {lo, %0}, u;\n\t}"
      : "=r"(hi) : "r"(a), "r"(b), "l"(c));
  return hi;
}

__device__ __forceinline__ unsigned long long wide(uint32_t a, int32_t b, unsigned long long c) {
  unsigned long long u;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(u) : "r"(a), "r"(b), "l"(c));
  return u;
}

template <int MODE>
__global__ void __launch_bounds__(NT, 2) probe(Tab tab, int iters, int n_rho, const uint32_t *edges,
                                               unsigned long long *cyc, uint32_t *sink) {
  extern __shared__ __align__(16) uint32_t sl[];
  __shared__ uint4 rowk[NP];
  __shared__ ulonglong2 rowq[NP];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 2 * NP * n_rho; i += NT) sl[i] = 0;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(sl));
  const int D = (n_rho - 1) / 2;
  const uint32_t koff = (1u << 14) + (static_cast<uint32_t>(D) << 15);
  if (tid < NP) {
    const uint32_t rb = sbase + tid * n_rho * 4;
    rowk[tid] = make_uint4(tab.c[tid], tab.s[tid], koff + (rb << 13), static_cast<uint32_t>(-tab.c[tid]));
    // wide: hi32 = floor(V/2^15) + rb/4 (row base folded in words)
    const unsigned long long k17 = (static_cast<unsigned long long>(koff) << 17) +
                                   (static_cast<unsigned long long>(rb >> 2) << 32);
    rowq[tid] = make_ulonglong2(static_cast<unsigned long long>(static_cast<long long>(tab.c[tid]) << 15),
                                k17);
  }
  __syncthreads();
  const uint32_t delta = NP * n_rho * 4;
  // synthetic edges: warp w, lane l -> x = 300 + l + (j & 1), y = 200 + 7*w + j
  uint32_t xs[EPL], ys[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    const uint32_t e = edges[(warp & 15) * 32 * EPL + j * 32 + lane];
    xs[j] = MODE == 0 ? (e & 0xFFFFu) : (e & 0xFFFFu) * 4u;
    ys[j] = MODE == 0 ? (e >> 16) : (e >> 16) * 4u;
  }
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 2
    for (int r = 0; r < NP; ++r) {
      if (MODE == 0) {
        const uint4 k = rowk[r];
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          const uint32_t q = ys[j] * k.y + k.z;
          red_add(((xs[j] * k.x + q) >> 13) & ~3u);
          red_add((((xs[j] * k.w + q) >> 13) & ~3u) + delta);
        }
      } else {
        const ulonglong2 k = rowq[r];
        const int32_t c15 = static_cast<int32_t>(k.x), s15 = tab.s[r] << 15;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          const unsigned long long Q = wide(ys[j], s15, k.y);
          red_add(wide_hi(xs[j], c15, Q) << 2);
          red_add((wide_hi(xs[j], -c15, Q) << 2) + delta);
        }
      }
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  uint32_t s = 0;
  for (int i = tid; i < 2 * NP * n_rho; i += NT) s += sl[i] * (i + 1);
  sink[blockIdx.x * NT + tid] = s;
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int n_rho = 2939;
  Tab tab;
  for (int i = 0; i < NP; ++i) {
    const double th = M_PI * (i * 11 + 3) / 180.0;
    tab.c[i] = static_cast<int>(floor(cos(th) * 32768.0 + 0.5));
    tab.s[i] = static_cast<int>(floor(sin(th) * 32768.0 + 0.5));
  }
  const int smem = 2 * NP * n_rho * 4 + 16;
  unsigned long long *cyc;
  uint32_t *sink, *h0, *h1, *edges;
  {
    uint32_t he[16 * 32 * EPL];
    for (int w = 0; w < 16; ++w)
      for (int j = 0; j < EPL; ++j)
        for (int l = 0; l < 32; ++l)
          he[w * 32 * EPL + j * 32 + l] = ((200u + 7 * w + j) << 16) | (300u + l + (j & 1));
    cudaMalloc(&edges, sizeof(he));
    cudaMemcpy(edges, he, sizeof(he), cudaMemcpyHostToDevice);
  }
  const int grid = 2 * sms;
  cudaMalloc(&cyc, grid * 8);
  cudaMalloc(&sink, grid * NT * 4);
  h0 = new uint32_t[grid * NT];
  h1 = new uint32_t[grid * NT];
  cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 64;
  for (int mode = 0; mode < 2; ++mode) {
    auto k = mode == 0 ? probe<0> : probe<1>;
    k<<<grid, NT, smem>>>(tab, 2, n_rho, edges, cyc, sink);
    k<<<grid, NT, smem>>>(tab, iters, n_rho, edges, cyc, sink);
    cudaDeviceSynchronize();
    unsigned long long h[4096];
    cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(mode == 0 ? h0 : h1, sink, grid * NT * 4, cudaMemcpyDeviceToHost);
    double mc = 0;
    for (int i = 0; i < grid; ++i) mc += h[i];
    mc /= grid;
    // two CTAs share an SM: ATOMS of both over one CTA's cycles
    const double atoms_per_cta = (NT / 32.0) * iters * NP * EPL * 2;
    printf("mode %d (%s): %.3f warp-ATOMS/clk/SM\n", mode, mode == 0 ? "shift" : "wide",
           2 * atoms_per_cta / mc);
  }
  int diff = 0;
  for (int i = 0; i < grid * NT; ++i) diff += h0[i] != h1[i];
  printf("checksums differ in %d threads; status %s\n", diff,
         cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
