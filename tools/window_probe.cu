// Cycle cost of the fused peak kernel's window test (ld_peaks.cu
// warp_window_max, copied into window_probe_body.cuh) on a cfg5-sized
// accumulator (1024 x 11587), window 21 x 233 around a passing cell, by one
// warp: cold (first touch) and warm, and with 1..32 warps testing at once.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Itools -o build/window_probe tools/window_probe.cu
#include <cstdio>
#include <cstdint>
#include "window_probe_body.cuh"

__global__ void probe(const uint32_t *A, int64_t ncells, int n_theta, int n_rho, int nw,
                      long long *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp >= nw) return;
  const int t = 500 + 3 * warp, r = 5000 + 40 * warp;
  long long c[3];
  bool ok = true;
  for (int rep = 0; rep < 3; ++rep) {
    const long long t0 = clock64();
    ok &= warp_window_max<4, false>(A, ncells, n_theta, n_rho, t, r, 1000u, 10, 116, lane);
    c[rep] = clock64() - t0;
  }
  if (lane == 0) {
    out[warp * 4 + 0] = c[0];
    out[warp * 4 + 1] = c[1];
    out[warp * 4 + 2] = c[2];
    out[warp * 4 + 3] = ok;
  }
}

int main() {
  const int nt = 1024, nr = 11587;
  const int64_t n = (int64_t)nt * nr;
  uint32_t *A;
  cudaMalloc(&A, n * 4);
  cudaMemset(A, 0, n * 4);
  long long *out, h[128];
  cudaMalloc(&out, sizeof(h));
  for (int nw : {1, 4, 32}) {
    // centre cells = 1000 (passing), everything else 0 (set per warp)
    cudaMemset(A, 0, n * 4);
    for (int w = 0; w < nw; ++w) {
      uint32_t v = 1000;
      cudaMemcpy(A + (int64_t)(500 + 3 * w) * nr + 5000 + 40 * w, &v, 4, cudaMemcpyHostToDevice);
    }
    probe<<<1, 32 * nw>>>(A, n, nt, nr, nw, out);
    cudaMemcpy(h, out, sizeof(long long) * 4 * nw, cudaMemcpyDeviceToHost);
    printf("warps=%2d  warp0: cold %6lld  warm %6lld %6lld  ok=%lld   last warp: %6lld %6lld\n", nw,
           h[0], h[1], h[2], h[3], h[4 * (nw - 1)], h[4 * (nw - 1) + 1]);
  }
  return 0;
}
