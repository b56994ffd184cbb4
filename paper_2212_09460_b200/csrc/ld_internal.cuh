// ld_internal.cuh -- shared declarations of the libld.so translation units.
// Product code only: nothing here is shared with oracle/.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <utility>

#include "../../include/ld.h"

namespace ld {

// ---------------------------------------------------------------------------
// B1: fused Sobel + binarize + compaction (ld_sobel.cu)
// ---------------------------------------------------------------------------
constexpr int SB_BOX_W = 256;       // TMA box width in bytes (hardware max 256)
constexpr int SB_HALO_L = 16;       // box starts 16 columns left of the tile
constexpr int SB_CHUNKS = 14;       // 16-px output chunks per tile row
constexpr int SB_TILE_W = SB_CHUNKS * 16;  // 224 output columns per tile
constexpr int SB_STRIPS = 16;       // thread strips per tile (vertical)
constexpr int SB_THREADS = SB_CHUNKS * SB_STRIPS;  // 224 = 7 consumer warps
#ifndef LD_SOBEL_CAP
#define LD_SOBEL_CAP 1024
#endif
constexpr int SB_STAGE_CAP = LD_SOBEL_CAP;  // per-warp edge staging buffer (uint32 entries)

// launch configuration: SR output rows per strip (tile height 16*SR), TMA ring
// depth, CTAs per SM, per-warp edge staging entries
struct SobelCfg {
  int sr, stages, ctas_per_sm;
  int cap = SB_STAGE_CAP;  // per-warp edge staging entries (0: direct global stores)
};
// rows = output rows owned, frames = batch, sms = SM count
SobelCfg sobel_cfg(int width, int rows, int frames, int sms);

struct SobelParams {
  int32_t width, height;
  int32_t row_begin, row_end;  // owned rows (global)
  int32_t ry0;                 // global row of tensor row 0 = max(row_begin-1, 0)
  int32_t tiles_x, tiles_y, tiles_per_frame, n_tiles;
  int32_t batch;
  int32_t sr;                  // output rows per thread strip (sobel_cfg; tile height 16 * sr)
  int32_t t2;                  // ceil(T/2) clamped to [0, 766]
  int32_t zero_pad;            // LD_FLAG_ZERO_PAD: filter the border on a zero-padded image
  uint8_t *binary;
  int64_t bin_pitch, bin_frame_stride;
  uint32_t *edges;
  int64_t edge_stride;
  uint32_t *counts;
};

cudaError_t launch_sobel(const CUtensorMap &tmap, const SobelParams &p, int sm_count,
                         cudaStream_t stream);

// ---------------------------------------------------------------------------
// B3: theta-band shared-memory Hough voting (ld_hough.cu)
// ---------------------------------------------------------------------------
struct TrigTable {
  int32_t c[LD_MAX_THETA];
  int32_t s[LD_MAX_THETA];
};

constexpr int LD_MAX_THETA_F64 = 1024;  // double tables are passed by value (2 x 8 KB)
struct TrigTableF64 {
  double c[LD_MAX_THETA_F64];
  double s[LD_MAX_THETA_F64];
};

struct HoughParams {
  const uint32_t *edges;
  const uint32_t *counts;
  int64_t edge_stride;
  int32_t batch;
  int32_t n_theta, n_rho;
  int32_t rows_per_band, n_bands;  // paired kernel: pairs per band, bands
  int32_t n_pairs;                 // paired kernel (NEXT 2): theta pairs (t, n_theta - t)
  int32_t koff;  // 2^14 + (D << 15): rho_bin = (x*C + y*S + koff) >> 15
  uint32_t *acc;
  uint32_t *hint_hdr;            // nullable: peak-hint header (written by CTA (0, 0))
  unsigned long long *hint_keys;  // [batch][n_bands][warps per CTA] per-warp maxima
  uint32_t *segmax;              // [batch][n_seg] maxima of the accumulator's 1 KB chunks
  int32_t n_seg;                 // chunks per frame (seg_count)
};

// Peak-hint buffer layout (ld_hough_accumulate_hint / ld_hough_peaks_hinted):
// a 64-byte header {magic, batch, n_theta, n_rho, n_bands, keys per band,
// n_seg, acc address lo, hi, 0...}, the per-warp maximum keys
// ([batch][n_bands][keys per band], capacity batch * n_theta *
// HINT_MAX_RANGES), then the chunk maxima [batch][n_seg] (DESIGN R25, R30):
// chunk q of frame f covers the SEG_BYTES-aligned global bytes
// [(c0 + q) * SEG_BYTES, +SEG_BYTES), c0 = (frame start address) / SEG_BYTES;
// the entry is the maximum of the frame's counters in the chunk (0 if none).
constexpr uint32_t HINT_MAGIC = 0x3248444Cu;  // "LDH2"
constexpr int HINT_HDR_BYTES = 64;
constexpr int SEG_BYTES = 1024;  // accumulator bytes per chunk maximum (256 counters)
// chunks a frame of n_cells counters can touch at any 4-byte-aligned start
__host__ __device__ constexpr int seg_count(int64_t n_cells) {
  return static_cast<int>((n_cells * 4 + SEG_BYTES - 1) / SEG_BYTES) + 1;
}
constexpr int HINT_MAX_RANGES = 32;  // ranges per band (warps of a 1024-thread CTA)

constexpr int HV_THREADS = 1024;  // threads per SM; a CTA has HV_THREADS / CTAS of them
constexpr int HV_MAX_ROWS = 256;

// CTAs per SM: 2 (half the shared memory each, so one CTA's prologue and
// write-out overlap the other's voting) when a band then still holds >= 8
// rows, else 1.  Returns 0 if a single row does not fit.
int hough_plan(int n_theta, int n_rho, size_t smem_optin, int *ctas, int *rows_per_band,
               int *n_bands, size_t *smem_bytes);
cudaError_t launch_hough(const HoughParams &p, const TrigTable &trig, int ctas, size_t smem_bytes,
                         cudaStream_t stream);
// SPEC float64 trig mode (NEXT 4, ld_hough_f64.cu): same planning as hough_plan.
cudaError_t launch_hough_f64(const HoughParams &p, const TrigTableF64 &trig, int ctas,
                             size_t smem_bytes, cudaStream_t stream);
// Half-angle paired voting (NEXT 2, Eq. 4-5): valid when the table is
// symmetric, C[n-t] = -C[t] and S[n-t] = S[t] for 0 < t < n (checked on the
// host).  Pair p = (t = p, n - t); p = 0 and p = n/2 (n even) have no partner
// and vote their mirror into a scratch row.  Same planning contract as
// hough_plan, in pairs.
int hough_pair_count(int n_theta);
int hough_plan_pairs(int n_theta, int n_rho, size_t smem_optin, int *ctas, int *pairs_per_band,
                     int *n_bands, size_t *smem_bytes);
// cluster > 1: the band's edges split over a thread-block cluster of that many
// CTAs whose shared-memory copies are summed over DSMEM (single frames);
// hough_cluster_size picks it (1 = no cluster).
int hough_cluster_size(int batch, int n_bands, int ctas, int sm_count);
cudaError_t launch_hough_pairs(const HoughParams &p, const TrigTable &trig, int ctas,
                               size_t smem_bytes, cudaStream_t stream, int cluster = 1);

// ---------------------------------------------------------------------------
// B4: peaks (ld_peaks.cu)
// ---------------------------------------------------------------------------
constexpr int PK_THREADS = 512;
constexpr int PK_ROWS = 4;         // theta rows per band CTA (generic kernel)
constexpr int PT_TR = 16;          // theta rows per tile (tiled kernel)
constexpr int PT_MAX_THREADS = 512;
constexpr int PT_MAX_HT = 12;      // largest half_theta with a tiled instance

struct PeaksParams {
  const uint32_t *acc;
  int32_t batch, n_theta, n_rho;
  int32_t half_theta, half_rho;
  uint32_t floor_votes;  // max(1, min_votes)
  int32_t k;
  int32_t n_units;                // tiles (tiled kernel) or bands (generic) per frame
  int32_t tch, tc, tiles_t, tiles_r;  // tiled kernel geometry
  int32_t st_nt, st_sw, st_strips, st_tb, st_chunks, st_buf;  // streaming kernel geometry
  unsigned long long *band_keys;  // [batch][n_units][k]
  uint32_t *gtau;                 // [batch] per-frame running k-th candidate value (stream kernel)
  int32_t cand_t0, cand_t1;       // candidate rows [cand_t0, cand_t1) (windows read every row)
  int32_t theta_offset;           // added to the row index in keys and reported theta bins
  const uint32_t *hint_hdr;       // nullable: peak hint (unrestricted searches only)
  const unsigned long long *hint_keys;
  const uint32_t *segmax;         // hint's chunk maxima [batch][n_seg] (sparse path)
  int32_t n_seg;
  uint32_t *resolved;             // [batch] 1 = the fused hinted search wrote this frame's peaks
  unsigned long long *diag;       // [batch][PF_DIAG] diagnostics (LD_PF_STATS builds)
  uint32_t *self_hdr = nullptr;   // workspace hint of the accumulator itself (no hint given)
  unsigned long long *self_keys = nullptr;
  uint32_t *self_segmax = nullptr;
  ld_peak *peaks;
  int32_t *n_peaks;
};
constexpr int SP_CAP = 2048;      // fused hinted search: candidate keys per frame
constexpr int PF_DIAG = 16;       // diagnostics words per frame in the peaks workspace

// Peaks workspace: byte offsets of its parts
struct PeaksLayout {
  size_t gtau, resolved, diag, keys, self_hdr, self_keys, self_segmax, total;
};
PeaksLayout peaks_layout(int batch, int n_theta, int n_rho, int k);
size_t peaks_workspace_bytes(int batch, int n_theta, int n_rho, int k);
// flags: LD_PEAKS_* of ld.h
cudaError_t launch_peaks(const PeaksParams &p, uint32_t flags, cudaStream_t stream);
// the peak hint of an existing accumulator into header, keys and chunk maxima
cudaError_t launch_hint_from_acc(const uint32_t *acc, int batch, int n_theta, int n_rho,
                                 int cand_t0, int cand_t1, uint32_t *hdr,
                                 unsigned long long *keys, uint32_t *segmax, cudaStream_t stream);
size_t hint_self_keys_bytes(int batch, int n_theta, int n_rho);

// ---------------------------------------------------------------------------
// NEXT 3: lanes module (ld_lanes.cu)
// ---------------------------------------------------------------------------
struct NmsState {
  unsigned long long best;  // arg-max key of the current round
  uint32_t npicks;
  uint32_t thr;             // eligibility threshold (0 until the first pick)
  uint32_t done;
  uint32_t pad;
};

struct NmsParams {
  const uint32_t *acc;
  int32_t batch, n_theta, n_rho, half_theta, half_rho, k;
  uint32_t floor_votes, ratio_num, ratio_den;
  NmsState *state;       // [batch]
  uint32_t *bitmap;      // [batch][bitmap_words] suppression bits
  int64_t bitmap_words;
  ld_peak *peaks;
  int32_t *n_peaks;
};
cudaError_t launch_nms(const NmsParams &p, cudaStream_t stream);

struct LanesParams {
  const ld_peak *peaks;   // [batch][k]
  const int32_t *n_peaks;  // [batch]
  int32_t batch, k, width, height, n_theta, rho_offset;
  ld_segment *lines;       // peak_to_line: [batch][k]
  int32_t *hit;            // [batch][k]
  const uint8_t *binary;   // extract_segments: [batch] frames of [height][bin_pitch]
  int64_t bin_pitch, bin_frame_stride;
  int32_t fill_gap, min_len, max_segs;
  ld_segment *segs;        // [batch][k][max_segs]
  int32_t *n_segs;         // [batch][k]
};
cudaError_t launch_peak_lines(const LanesParams &p, const TrigTable &trig, cudaStream_t stream);
cudaError_t launch_extract_segments(const LanesParams &p, const TrigTable &trig,
                                    cudaStream_t stream);

// ---------------------------------------------------------------------------
// Multi-GPU helpers (ld_dist.cu)
// ---------------------------------------------------------------------------
cudaError_t launch_edges_to_bitmask(const uint32_t *edges, const uint32_t *count, int width,
                                    int row_begin, int rows, uint32_t *bits, int sm_count,
                                    cudaStream_t stream);
cudaError_t launch_bitmask_to_edges(const uint32_t *bits, int width, int n_blocks,
                                    const int32_t *row_begin, const int32_t *rows,
                                    int block_stride_rows, uint32_t *edges, int64_t capacity,
                                    uint32_t *count, cudaStream_t stream);
cudaError_t launch_merge_peak_lists(const ld_peak *peaks, const int32_t *n_peaks, int n_lists,
                                    int k, int n_rho, ld_peak *out, int32_t *n_out,
                                    cudaStream_t stream);

// ---------------------------------------------------------------------------
// B5: shared-memory atomic microbenchmark (ld_hough.cu)
// ---------------------------------------------------------------------------
cudaError_t launch_smem_atomic_bench(int mode, int iters, int grid, uint32_t *scratch,
                                     cudaStream_t stream);

// launch counter of the current host thread (ld_api.cu)
void note_launch(int n = 1);

// Per-device, per-kernel "max dynamic shared memory" attribute, set once:
// std::call_once per (device, kernel) slot -- thread-safe, no racy flags.
struct AttrOnce {
  std::once_flag once[64];
  cudaError_t err[64] = {};
};

// bytes >= 0: that many bytes; bytes < 0: -bytes minus the kernel's static
// shared memory (the largest request a CTA of that kernel can make).
template <typename K>
static inline cudaError_t ensure_smem_attr(AttrOnce &a, K kern, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::call_once(a.once[dev & 63], [&]() {
    int b = bytes;
    if (b < 0) {
      cudaFuncAttributes fa;
      const cudaError_t r = cudaFuncGetAttributes(&fa, kern);
      if (r != cudaSuccess) {
        a.err[dev & 63] = r;
        return;
      }
      b = -bytes - static_cast<int>(fa.sharedSizeBytes);
    }
    a.err[dev & 63] = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  });
  return a.err[dev & 63];
}

// One kernel launch of the detect path: programmatic stream serialization
// (the kernel may start while the previous kernel of the stream finishes; it
// calls pdl_wait before reading that kernel's outputs) and, for cluster > 1,
// a thread-block cluster of that many CTAs along x.  Counts the launch.
#ifndef LD_PDL
#define LD_PDL 1
#endif
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                    cudaStream_t stream, int cluster, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (LD_PDL) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = static_cast<unsigned>(cluster);
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  note_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// (bar_s: the barrier's shared-memory address, for loops that hoist it)
__device__ __forceinline__ void mbar_arrive_s(uint32_t bar_s) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_s) : "memory");
}

__device__ __forceinline__ void mbar_wait_s(uint32_t bar_s, uint32_t parity) {
  // try_wait with a suspend-time hint: the waiting thread sleeps in hardware
  // until the phase completes (or the hint expires) instead of spinning on
  // the issue slots other warps need
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "LD_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 0x989680;\n\t"
      "@!p bra LD_WAIT_%=;\n}" ::"r"(bar_s),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  mbar_wait_s(smem_u32(bar), parity);
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// Programmatic dependent launch (the kernels of one detect step are launched
// with cudaLaunchAttributeProgrammaticStreamSerialization, launch_ex below):
// every CTA lets the next kernel of the stream launch as soon as it runs
// (pdl_launch_dependents: the next grid then fills the SMs this one frees in
// its last wave and runs its own set-up), and waits for the previous kernel
// to complete and flush (pdl_wait) before it reads that kernel's outputs.
// Both are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// an early trigger in every CTA (experiment; default: the implicit trigger
// at CTA exit, so waiting dependents never hold SM resources other streams'
// kernels could use)
#ifndef LD_PDL_EARLY
#define LD_PDL_EARLY 0
#endif
#if LD_PDL_EARLY
#define LD_PDL_TRIGGER() pdl_launch_dependents()
#else
#define LD_PDL_TRIGGER() ((void)0)
#endif

// shared-memory writes of this thread -> visible to the async proxy (bulk copies)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// this thread's committed bulk copies have finished READING shared memory
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ void red_shared_add(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

}  // namespace ld
