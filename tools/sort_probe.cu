// Cycle cost of the fused peak kernel's block sort (ld_peaks.cu
// block_sort_desc, copied here for the probe) for n2 keys and NT threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/sort_probe tools/sort_probe.cu
#include <cstdio>
#include <cstdint>
typedef unsigned long long u64;
#define PROBE 1
#include "sort_probe_body.cuh"

template <int NT, int S>
__global__ void __launch_bounds__(NT, 1024 / NT) probe(int n2, long long *out, u64 *res) {
  __shared__ u64 a[2048];
  u64 x[S];
  for (int s = 0; s < S; ++s) {
    const int e = s * NT + threadIdx.x;
    x[s] = e < n2 ? (u64)((e * 2654435761u) % 100000u) << 32 | e : 0ull;
  }
  __syncthreads();
  long long t0 = clock64();
  block_sort_desc<NT, S>(a, n2, x);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  for (int i = threadIdx.x; i < n2; i += NT) res[i] = a[i];
}

int main() {
  long long *out;
  u64 *res;
  cudaMalloc(&out, 8);
  cudaMalloc(&res, 8 * 2048);
  for (int n2 : {32, 256, 512, 2048}) {
    long long c1 = 0, c2 = 0, h;
    for (int rep = 0; rep < 3; ++rep) {
      probe<1024, 2><<<1, 1024>>>(n2, out, res);
      cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
      c1 = h;
      probe<512, 4><<<1, 512>>>(n2, out, res);
      cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
      c2 = h;
    }
    u64 r[2048];
    cudaMemcpy(r, res, 8 * n2, cudaMemcpyDeviceToHost);
    int ok = 1;
    for (int i = 1; i < n2; ++i) ok &= r[i - 1] >= r[i];
    printf("n2=%4d  NT=1024: %6lld cycles   NT=512: %6lld cycles  sorted=%d\n", n2, c1, c2, ok);
  }
  return 0;
}
