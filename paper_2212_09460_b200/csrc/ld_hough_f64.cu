// ld_hough_f64.cu -- SPEC's float64 trig mode of the voting (SURVEY 8(f)
// NEXT 4, "a second, non-bit-exact-vs-Q15 workload"; DESIGN R29).
//
// Same theta-band shared-memory design as ld_hough.cu (hough_plan bands, a
// CTA per band, ATOMS into the band's slice, bulk write-out), with the
// caller's double-precision table instead of Q15:
//   r = x*cos[t] + y*sin[t]  (__dmul_rn twice, __dadd_rn: each rounded once,
//                             the oracle's exact operation order, no FMA)
//   rho = floor(r + 0.5) + D (cvt.rmi: floor in the conversion)
// The host proves the corner range with the same arithmetic (r is monotone
// in x and y under round-to-nearest), so no vote needs a bounds check.
#include "ld_internal.cuh"

namespace ld {

template <int EPL, bool FULL>
__device__ __forceinline__ void vote_block_f64(const uint32_t *el, uint32_t blk, uint32_t end,
                                               int lane, int nr, const double2 *cs,
                                               const uint32_t *rbase, uint32_t scratch) {
  double xs[EPL], ys[EPL];
  bool ok[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    const uint32_t e = blk + 32u * j + lane;
    ok[j] = FULL || e < end;
    const uint32_t q = ok[j] ? __ldg(el + e) : 0u;
    xs[j] = static_cast<double>(q & 0xFFFFu);
    ys[j] = static_cast<double>(q >> 16);
  }
#pragma unroll 2
  for (int r = 0; r < nr; ++r) {
    const double2 k = cs[r];
    const uint32_t b = rbase[r];  // row address + 4 D
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const double rr = __dadd_rn(__dmul_rn(xs[j], k.x), __dmul_rn(ys[j], k.y));
      const int q = __double2int_rd(__dadd_rn(rr, 0.5));
      const uint32_t a = b + (static_cast<uint32_t>(q) << 2);
      red_shared_add(FULL || ok[j] ? a : scratch, 1u);
    }
  }
}

template <int CTAS>
__global__ void __launch_bounds__(HV_THREADS / CTAS, CTAS)
    hough_vote_f64_kernel(const HoughParams p, const __grid_constant__ TrigTableF64 trig) {
  constexpr int NT = HV_THREADS / CTAS;
  constexpr int NWARPS = NT / 32;
  extern __shared__ __align__(16) uint32_t slice_raw[];
  __shared__ double2 cs[HV_MAX_ROWS];
  __shared__ uint32_t rbase[HV_MAX_ROWS];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int band = blockIdx.x;
  const int f = blockIdx.y;
  const int t0 = band * p.rows_per_band;
  const int nr = min(p.rows_per_band, p.n_theta - t0);
  const int ncell = nr * p.n_rho;
  uint32_t *dst = p.acc + (static_cast<int64_t>(f) * p.n_theta + t0) * p.n_rho;
  const int mw = static_cast<int>((reinterpret_cast<uintptr_t>(dst) & 15u) >> 2);
  uint32_t *slice = slice_raw + mw;
  const uint32_t sbase = smem_u32(slice);
  const uint32_t row_bytes = static_cast<uint32_t>(p.n_rho) * 4u;
  const uint32_t d4 = static_cast<uint32_t>((p.n_rho - 1) / 2) * 4u;  // 4 D
  {
    uint4 *s4 = reinterpret_cast<uint4 *>(slice_raw);
    const int n4 = (mw + ncell + 3) >> 2;
    for (int i = tid; i < n4; i += NT) s4[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int i = tid; i < nr; i += NT) {
      cs[i] = make_double2(trig.c[t0 + i], trig.s[t0 + i]);
      rbase[i] = sbase + i * row_bytes + d4;
    }
  }
  __syncthreads();

  const uint32_t n_edges = p.counts[f];
  const uint32_t *el = p.edges + static_cast<int64_t>(f) * p.edge_stride;
  const uint32_t scratch = smem_u32(slice + ncell);
  uint32_t base = 0;
  for (; base + NWARPS * 32u * 8u <= n_edges; base += NWARPS * 32u * 8u)
    vote_block_f64<8, true>(el, base + warp * 32u * 8u, n_edges, lane, nr, cs, rbase, scratch);
  const uint32_t blk = base + static_cast<uint32_t>(warp) * (32u * 8u);
  if (blk < n_edges) vote_block_f64<8, false>(el, blk, n_edges, lane, nr, cs, rbase, scratch);
  __syncthreads();

  const int head = min((4 - mw) & 3, ncell);
  const int mid = ((ncell - head) >> 2) << 2;
  if (tid < head) dst[tid] = slice[tid];
  for (int i = head + mid + tid; i < ncell; i += NT) dst[i] = slice[i];
  if (tid == 0 && mid > 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + head),
                 "r"(smem_u32(slice + head)), "r"(static_cast<uint32_t>(mid) * 4u)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

static AttrOnce g_f64_attr[3];

cudaError_t launch_hough_f64(const HoughParams &p, const TrigTableF64 &trig, int ctas,
                             size_t smem_bytes, cudaStream_t stream) {
  auto kern = ctas == 2 ? hough_vote_f64_kernel<2> : hough_vote_f64_kernel<1>;
  const cudaError_t e = ensure_smem_attr(g_f64_attr[ctas], kern, -(227 * 1024 / ctas));
  if (e != cudaSuccess) return e;
  dim3 grid(p.n_bands, p.batch);
  kern<<<grid, HV_THREADS / ctas, smem_bytes, stream>>>(p, trig);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ld
