// Shared-memory atomic cost model probe (not part of libld.so).
//
// Each lane issues red.shared.add.u32 at  base + row*4096 + 4*off(lane)
// for 32 rows per unrolled group (immediate offsets: the SASS is pure ATOMS),
// with the lane offsets of a pattern:
//   0 distinct   off = l                    (32 addresses, 32 banks)
//   1 pairs      off = l/2                  (16 addresses, 2 lanes each)
//   2 quads      off = l/4                  (8 addresses, 4 lanes each)
//   3 same       off = 0                    (1 address; rows rotate)
//   4 conf2      off = l%16 + 32*(l/16)     (32 addresses, 2 per bank)
//   5 conf4      off = l%8  + 32*(l/8)      (32 addresses, 4 per bank)
//   6 half       off = l, lanes >= 16 idle  (16 active lanes)
//   7 span40     off = (l*40)/32            (32 addresses over 40 words: 8 banks 2-way)
// Prints warp-ATOMS per clock per SM (from clock64 in every CTA) and the
// event-timed lane rate.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o atoms_probe tools/atoms_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

// -DADD_VAL=65536: the increment of a 16-bit counter in a word's high half
// (SASS ATOMS.ADD with a register operand instead of ATOMS.POPC.INC)
#ifndef ADD_VAL
#define ADD_VAL 1
#endif
__device__ __forceinline__ void red_add(uint32_t a) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "n"(ADD_VAL) : "memory");
}

__global__ void probe(int mode, int iters, unsigned long long *cyc, uint32_t *sink) {
  extern __shared__ __align__(16) uint32_t buf[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int words = 32 * 1024;  // 128 KB: 32 rows of 4096 B
  for (int i = tid; i < words; i += blockDim.x) buf[i] = 0u;
  __syncthreads();
  int off;
  switch (mode) {
    case 0: off = lane; break;
    case 1: off = lane >> 1; break;
    case 2: off = lane >> 2; break;
    case 3: off = 0; break;
    case 4: off = (lane & 15) + 32 * (lane >> 4); break;
    case 5: off = (lane & 7) + 32 * (lane >> 3); break;
    case 6: off = lane; break;
    default: off = (lane * 40) / 32; break;
  }
  // spread warps over the row's 1024 words so different warps do not share
  // addresses (only the intra-warp pattern matters)
  const int w = tid >> 5;
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(buf)) +
                     4u * static_cast<uint32_t>((off + 128 * (w & 7)) & 1023);
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (mode != 6 || lane < 16) {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 32; ++j) red_add(a + j * 4096u);
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  if (tid < 32) {
    uint32_t s = 0;
    for (int i = tid; i < words; i += 32) s += buf[i];
    sink[blockIdx.x * 32 + tid] = s;
  }
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = 128 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long *cyc;
  uint32_t *sink;
  cudaMalloc(&cyc, sms * 8 * sizeof(unsigned long long));
  cudaMalloc(&sink, sms * 8 * 32 * 4);
  const char *names[] = {"distinct", "pairs", "quads", "same", "conf2", "conf4", "half16", "span40"};
  const int iters = 256;
  for (int threads : {1024, 512}) {
    for (int mode = 0; mode < 8; ++mode) {
      probe<<<sms, threads, smem>>>(mode, 8, cyc, sink);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      probe<<<sms, threads, smem>>>(mode, iters, cyc, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long h[1024];
      cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
      double mc = 0;
      for (int i = 0; i < sms; ++i) mc += h[i];
      mc /= sms;
      const double warp_atoms = (threads / 32.0) * iters * 32.0;  // per SM
      const double lanes = warp_atoms * (mode == 6 ? 16 : 32) * sms;
      printf("threads %4d  %-8s  %.3f warp-ATOMS/clk/SM   %.1f G lane-atomics/s  (%.3f ms)\n",
             threads, names[mode], warp_atoms / mc, lanes / (ms * 1e-3) / 1e9, ms);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
