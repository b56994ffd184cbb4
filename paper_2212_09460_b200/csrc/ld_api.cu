// ld_api.cu -- host side of libld.so: validation, geometry, TMA descriptor
// encoding, launch configuration, workspace layout and the C ABI of include/ld.h.
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "ld_internal.cuh"

#include <nvtx3/nvToolsExt.h>  // header-only: ranges cost nothing without a profiler

namespace ld {

static thread_local char g_err[512] = "";
static thread_local int g_launches = 0;

void note_launch(int n) { g_launches += n; }

static int fail(int status, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

static int cuda_fail(cudaError_t e, const char *what) {
  return fail(LD_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

struct DevInfo {
  bool ok = false;
  int sm_count = 0;
  int smem_optin = 0;
  int64_t l2 = 0;
  int major = 0, minor = 0;
};

static std::mutex g_mu;
static DevInfo g_dev[64];
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int device_info(DevInfo *out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_mu);
  DevInfo &d = g_dev[dev & 63];
  if (!d.ok) {
    cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    d.l2 = l2;
    cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&d.minor, cudaDevAttrComputeCapabilityMinor, dev);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    d.ok = true;
  }
  *out = d;
  if (d.major != 10 || d.minor != 0)
    return fail(LD_ERR_UNSUPPORTED, "device is sm_%d%d; libld.so is built for sm_100a only",
                d.major, d.minor);
  return LD_OK;
}

static int get_encoder() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_encode) return LD_OK;
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
    return fail(LD_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return LD_OK;
}

static int32_t rho_offset(int32_t w, int32_t h) {
  if (w < 1 || h < 1) return -1;
  const int64_t s = static_cast<int64_t>(w) * w + static_cast<int64_t>(h) * h;
  int64_t r = static_cast<int64_t>(std::sqrt(static_cast<double>(s)));
  while (r * r < s) ++r;
  while (r > 0 && (r - 1) * (r - 1) >= s) --r;
  return static_cast<int32_t>(r);
}

static bool aligned(const void *p, uintptr_t a) {
  return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0;
}

static int check_image(const uint8_t *gray, const ld_image *img) {
  if (!img) return fail(LD_ERR_INVALID_ARG, "img is NULL");
  if (!gray) return fail(LD_ERR_INVALID_ARG, "gray is NULL");
  if (img->width < 1 || img->height < 1 || img->width > LD_MAX_DIM || img->height > LD_MAX_DIM)
    return fail(LD_ERR_INVALID_ARG, "width/height %d x %d outside [1, %d]", img->width,
                img->height, LD_MAX_DIM);
  if (img->pitch < img->width || img->pitch % 16 != 0)
    return fail(LD_ERR_INVALID_ARG, "pitch %lld must be >= width and a multiple of 16",
                static_cast<long long>(img->pitch));
  if (img->batch < 1) return fail(LD_ERR_INVALID_ARG, "batch must be >= 1");
  if (img->row_begin < 0 || img->row_end > img->height || img->row_begin >= img->row_end)
    return fail(LD_ERR_INVALID_ARG, "rows [%d, %d) invalid for height %d", img->row_begin,
                img->row_end, img->height);
  const int ry0 = img->row_begin > 0 ? img->row_begin - 1 : 0;
  const int ry1 = img->row_end < img->height ? img->row_end + 1 : img->height;
  if (img->batch > 1 &&
      (img->frame_stride % 16 != 0 || img->frame_stride < static_cast<int64_t>(ry1 - ry0) * img->pitch))
    return fail(LD_ERR_INVALID_ARG, "frame_stride %lld must be a multiple of 16 and >= %lld",
                static_cast<long long>(img->frame_stride),
                static_cast<long long>(ry1 - ry0) * img->pitch);
  if (!aligned(gray, 16)) return fail(LD_ERR_INVALID_ARG, "gray must be 16-byte aligned");
  return LD_OK;
}

static int64_t max_edges_per_frame(const ld_image *img, uint32_t flags = 0) {
  const int64_t w2 = (flags & LD_FLAG_ZERO_PAD) ? img->width : (img->width > 2 ? img->width - 2 : 0);
  return static_cast<int64_t>(img->row_end - img->row_begin) * w2;
}

// Range proof (ld.h): |C|,|S| <= 32768 and the corner rho bins are in range.
static int check_trig(int32_t n_theta, const int32_t *c, const int32_t *s, int32_t w,
                      int32_t h, int32_t d) {
  if (n_theta < 1 || n_theta > LD_MAX_THETA)
    return fail(LD_ERR_INVALID_ARG, "n_theta %d outside [1, %d]", n_theta, LD_MAX_THETA);
  if (!c || !s) return fail(LD_ERR_INVALID_ARG, "trig table pointer is NULL");
  const int64_t n_rho = 2 * static_cast<int64_t>(d) + 1;
  const int64_t xs[2] = {0, w - 1}, ys[2] = {0, h - 1};
  for (int t = 0; t < n_theta; ++t) {
    if (c[t] < -32768 || c[t] > 32768 || s[t] < -32768 || s[t] > 32768)
      return fail(LD_ERR_RANGE, "trig entry %d (%d, %d) exceeds |32768|", t, c[t], s[t]);
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        const int64_t v = xs[a] * c[t] + ys[b] * s[t] + 16384 + (static_cast<int64_t>(d) << 15);
        const int64_t rho = v >> 15;  // v >= 0 is required too (floor of a negative)
        if (v < 0 || rho < 0 || rho >= n_rho)
          return fail(LD_ERR_RANGE, "theta bin %d sends corner (%lld, %lld) to rho bin %lld",
                      t, static_cast<long long>(xs[a]), static_cast<long long>(ys[b]),
                      static_cast<long long>(rho));
      }
  }
  return LD_OK;
}

// Half-angle pairing (NEXT 2) is exact iff the table is symmetric,
// C[n-t] = -C[t] and S[n-t] = S[t] for 0 < t < n, t != n/2; the unpaired rows
// (t = 0, t = n/2) also vote their mirror (-C[t], S[t]) into a scratch row,
// whose bins must pass the same corner range proof.
static bool pairable_trig(int32_t n_theta, const int32_t *c, const int32_t *s, int32_t w,
                          int32_t h, int32_t d) {
  for (int t = 1; t < n_theta; ++t)
    if (2 * t != n_theta && (c[n_theta - t] != -c[t] || s[n_theta - t] != s[t])) return false;
  const int64_t n_rho = 2 * static_cast<int64_t>(d) + 1;
  const int64_t xs[2] = {0, w - 1}, ys[2] = {0, h - 1};
  for (int t = 0; t < n_theta; t += (n_theta % 2 == 0 && n_theta > 1) ? n_theta / 2 : n_theta) {
    if (-static_cast<int64_t>(c[t]) > 32768) return false;
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        const int64_t v = -xs[a] * c[t] + ys[b] * s[t] + 16384 + (static_cast<int64_t>(d) << 15);
        if (v < 0 || (v >> 15) >= n_rho) return false;
      }
  }
  return true;
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// ---------------------------------------------------------------------------
static int sobel_impl(const uint8_t *gray, const ld_image *img, int32_t threshold,
                      uint32_t flags, uint8_t *binary, uint32_t *edge_xy, int64_t edge_stride,
                      uint32_t *edge_count, cudaStream_t stream) {
  DevInfo dev;
  int rc = device_info(&dev);
  if (rc) return rc;
  if ((rc = get_encoder())) return rc;

  const int W = img->width, H = img->height;
  const int ry0 = img->row_begin > 0 ? img->row_begin - 1 : 0;
  const int ry1 = img->row_end < H ? img->row_end + 1 : H;
  const int rows_read = ry1 - ry0;
  const int64_t fstride = img->batch > 1 ? img->frame_stride
                                         : static_cast<int64_t>(rows_read) * img->pitch;

  CUtensorMap tmap;
  cuuint64_t gdim[3] = {static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(rows_read),
                        static_cast<cuuint64_t>(img->batch)};
  cuuint64_t gstride[2] = {static_cast<cuuint64_t>(img->pitch), static_cast<cuuint64_t>(fstride)};
  const SobelCfg cfg = sobel_cfg(W, img->row_end - img->row_begin, img->batch, dev.sm_count);
  const int tile_h = cfg.sr * SB_STRIPS;
  cuuint32_t box[3] = {SB_BOX_W, static_cast<cuuint32_t>(tile_h + 2), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = g_encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t *>(gray),
                         gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(LD_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", cr);

  SobelParams p;
  p.width = W;
  p.height = H;
  p.row_begin = img->row_begin;
  p.row_end = img->row_end;
  p.ry0 = ry0;
  p.tiles_x = (W + SB_TILE_W - 1) / SB_TILE_W;
  p.tiles_y = (img->row_end - img->row_begin + tile_h - 1) / tile_h;
  p.tiles_per_frame = p.tiles_x * p.tiles_y;
  p.sr = cfg.sr;
  const int64_t n_tiles = static_cast<int64_t>(p.tiles_per_frame) * img->batch;
  if (n_tiles > (1ll << 30)) return fail(LD_ERR_INVALID_ARG, "batch too large");
  p.n_tiles = static_cast<int32_t>(n_tiles);
  p.batch = img->batch;
  int t2 = threshold <= 0 ? 0 : static_cast<int>((static_cast<int64_t>(threshold) + 1) / 2);
  // LD_FLAG_CLAMP_255: min(|G|, 255) >= T is |G| >= T for T <= 255
  // and never true above it (t2 = 766 exceeds max |A|, |B| = 765)
  if ((flags & LD_FLAG_CLAMP_255) && threshold > 255) t2 = 766;
  p.t2 = t2 > 766 ? 766 : t2;
  p.zero_pad = (flags & LD_FLAG_ZERO_PAD) ? 1 : 0;
  p.binary = binary;
  p.bin_pitch = img->pitch;
  p.bin_frame_stride = static_cast<int64_t>(img->row_end - img->row_begin) * img->pitch;
  p.edges = edge_xy;
  p.edge_stride = edge_stride;
  p.counts = edge_count;

  cudaError_t e = cudaMemsetAsync(edge_count, 0, sizeof(uint32_t) * img->batch, stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(edge_count)");
  e = launch_sobel(tmap, p, dev.sm_count, stream);
  if (e != cudaSuccess) return cuda_fail(e, "sobel_binarize_compact_kernel launch");
  return LD_OK;
}

static size_t hint_keys_bytes(int32_t batch, int32_t n_theta) {
  // the band count never exceeds n_theta
  return sizeof(unsigned long long) * static_cast<size_t>(batch) * n_theta * HINT_MAX_RANGES;
}

static int32_t n_seg_of(int32_t n_theta, int32_t n_rho) {
  return seg_count(static_cast<int64_t>(n_theta) * n_rho);
}

static size_t hint_bytes(int32_t batch, int32_t n_theta, int32_t n_rho) {
  return HINT_HDR_BYTES + hint_keys_bytes(batch, n_theta) +
         sizeof(uint32_t) * static_cast<size_t>(batch) * n_seg_of(n_theta, n_rho);
}

static int hough_impl(const uint32_t *edge_xy, const uint32_t *edge_count, int64_t edge_stride,
                      int32_t batch, int32_t width, int32_t height, int32_t n_theta,
                      const int32_t *cos_q15, const int32_t *sin_q15, uint32_t *acc,
                      cudaStream_t stream, void *hint = nullptr, uint32_t flags = 0) {
  DevInfo dev;
  int rc = device_info(&dev);
  if (rc) return rc;
  const int32_t d = rho_offset(width, height);
  if ((rc = check_trig(n_theta, cos_q15, sin_q15, width, height, d))) return rc;
  const int n_rho = 2 * d + 1;
  int ctas = 1, rpb = 0, n_bands = 0;
  size_t smem = 0;
  const bool paired = !(flags & LD_VOTE_PLAIN) &&
                      pairable_trig(n_theta, cos_q15, sin_q15, width, height, d) &&
                      hough_plan_pairs(n_theta, n_rho, static_cast<size_t>(dev.smem_optin), &ctas,
                                       &rpb, &n_bands, &smem);
  if (!paired &&
      !hough_plan(n_theta, n_rho, static_cast<size_t>(dev.smem_optin), &ctas, &rpb, &n_bands, &smem))
    return fail(LD_ERR_UNSUPPORTED, "one accumulator row (%d bins) exceeds shared memory", n_rho);
// Launches too small to fill the GPU (single frames): one pair per band, so
// the frame's bands alone give more CTAs -- each streams the whole edge list
// for two rows, with no cluster reduction (cfg2 voting 18.4 -> 14.3 us, cfg1
// 11.7 -> 5.6 us; cfg2 frames/s +13 % with 4 streams; DESIGN 6.2).  The
// cluster split (below) still applies when even one-pair bands are too few.
#ifndef LD_HV_SMALL_PPB
#define LD_HV_SMALL_PPB 1
#endif
  if (LD_HV_SMALL_PPB > 0 && paired && 2 * static_cast<int64_t>(batch) * n_bands <= dev.sm_count &&
      rpb > LD_HV_SMALL_PPB) {
    rpb = LD_HV_SMALL_PPB;
    n_bands = (hough_pair_count(n_theta) + rpb - 1) / rpb;
    smem = ((static_cast<size_t>(rpb) * n_rho * 8u + 15) / 16) * 16 + 64;
  }
  static thread_local TrigTable trig;  // 16 KB: keep it off the stack
  memcpy(trig.c, cos_q15, sizeof(int32_t) * n_theta);
  memcpy(trig.s, sin_q15, sizeof(int32_t) * n_theta);
  HoughParams p;
  p.edges = edge_xy;
  p.counts = edge_count;
  p.edge_stride = edge_stride;
  p.batch = batch;
  p.n_theta = n_theta;
  p.n_rho = n_rho;
  p.rows_per_band = rpb;
  p.n_bands = n_bands;
  p.koff = 16384 + (d << 15);
  p.acc = acc;
  p.hint_hdr = static_cast<uint32_t *>(hint);
  p.hint_keys = hint ? reinterpret_cast<unsigned long long *>(static_cast<char *>(hint) + HINT_HDR_BYTES)
                     : nullptr;
  p.segmax = hint ? reinterpret_cast<uint32_t *>(static_cast<char *>(hint) + HINT_HDR_BYTES +
                                                 hint_keys_bytes(batch, n_theta))
                  : nullptr;
  p.n_seg = n_seg_of(n_theta, n_rho);
  p.n_pairs = paired ? hough_pair_count(n_theta) : 0;
  if (p.segmax) {  // shared chunks are combined with atomicMax (ld_hough.cu summarize_block)
    cudaError_t e = cudaMemsetAsync(p.segmax, 0, sizeof(uint32_t) * static_cast<size_t>(batch) * p.n_seg,
                                    stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(segmax)");
  }
  const int cluster = paired && !(flags & LD_VOTE_NO_CLUSTER)
                          ? hough_cluster_size(batch, n_bands, ctas, dev.sm_count) : 1;
  cudaError_t e = paired ? launch_hough_pairs(p, trig, ctas, smem, stream, cluster)
                         : launch_hough(p, trig, ctas, smem, stream);
  if (e != cudaSuccess) return cuda_fail(e, "hough_vote_kernel launch");
  return LD_OK;
}

static int peaks_impl(const uint32_t *acc, int32_t batch, int32_t n_theta, int32_t n_rho,
                      int32_t half_theta, int32_t half_rho, uint32_t min_votes, int32_t k,
                      ld_peak *peaks, int32_t *n_peaks, void *workspace, size_t ws_bytes,
                      cudaStream_t stream, int32_t cand_t0 = 0, int32_t cand_t1 = -1,
                      int32_t theta_offset = 0, const void *hint = nullptr, uint32_t flags = 0) {
  PeaksParams p;
  p.acc = acc;
  p.batch = batch;
  p.n_theta = n_theta;
  p.n_rho = n_rho;
  p.half_theta = half_theta;
  p.half_rho = half_rho;
  p.floor_votes = min_votes > 1 ? min_votes : 1u;
  p.k = k;
  p.n_units = 0;
  p.cand_t0 = cand_t0;
  p.cand_t1 = cand_t1 < 0 ? n_theta : cand_t1;
  p.theta_offset = theta_offset;
  p.hint_hdr = static_cast<const uint32_t *>(hint);
  p.hint_keys = hint ? reinterpret_cast<const unsigned long long *>(static_cast<const char *>(hint) +
                                                                    HINT_HDR_BYTES)
                     : nullptr;
  p.segmax = hint ? reinterpret_cast<const uint32_t *>(static_cast<const char *>(hint) +
                                                       HINT_HDR_BYTES + hint_keys_bytes(batch, n_theta))
                  : nullptr;
  p.n_seg = n_seg_of(n_theta, n_rho);
  const PeaksLayout W = peaks_layout(batch, n_theta, n_rho, k);
  char *ws = static_cast<char *>(workspace);
  p.gtau = reinterpret_cast<uint32_t *>(ws + W.gtau);
  p.resolved = reinterpret_cast<uint32_t *>(ws + W.resolved);
  p.diag = reinterpret_cast<unsigned long long *>(ws + W.diag);
  p.self_hdr = reinterpret_cast<uint32_t *>(ws + W.self_hdr);
  p.self_keys = reinterpret_cast<unsigned long long *>(ws + W.self_keys);
  p.self_segmax = reinterpret_cast<uint32_t *>(ws + W.self_segmax);
  p.band_keys = reinterpret_cast<unsigned long long *>(ws + W.keys);
  p.peaks = peaks;
  p.n_peaks = n_peaks;
  (void)ws_bytes;
  cudaError_t e = launch_peaks(p, flags, stream);
  if (e != cudaSuccess) return cuda_fail(e, "peaks kernels launch");
  return LD_OK;
}

static int check_peaks_args(const uint32_t *acc, int32_t batch, int32_t n_theta, int32_t n_rho,
                            int32_t half_theta, int32_t half_rho, int32_t k, const ld_peak *peaks,
                            const int32_t *n_peaks) {
  if (!acc || !peaks || !n_peaks) return fail(LD_ERR_INVALID_ARG, "NULL acc/peaks/n_peaks");
  if (batch < 1 || n_theta < 1 || n_theta > LD_MAX_THETA || n_rho < 1)
    return fail(LD_ERR_INVALID_ARG, "bad accumulator shape [%d][%d][%d]", batch, n_theta, n_rho);
  if (static_cast<int64_t>(n_theta) * n_rho >= (1ll << 32) - 1)
    return fail(LD_ERR_INVALID_ARG, "accumulator too large for the 32-bit cell index");
  if (half_theta < 0 || half_rho < 0) return fail(LD_ERR_INVALID_ARG, "negative window");
  if (k < 1 || k > LD_MAX_K) return fail(LD_ERR_INVALID_ARG, "k %d outside [1, %d]", k, LD_MAX_K);
  return LD_OK;
}


struct DetectLayout {
  size_t counts_off, edges_off, acc_off, hint_off, peaks_off, total;
  int64_t edge_stride;
};

static DetectLayout detect_layout(const ld_image *img, int32_t n_theta, int32_t k, bool acc_ws) {
  DetectLayout L;
  const int64_t me = max_edges_per_frame(img, LD_FLAG_ZERO_PAD);  // any flags
  L.edge_stride = static_cast<int64_t>(align_up(static_cast<size_t>(me > 0 ? me : 1), 4));
  const int32_t d = rho_offset(img->width, img->height);
  const size_t acc_bytes = static_cast<size_t>(img->batch) * n_theta * (2 * static_cast<size_t>(d) + 1) * 4;
  size_t off = 0;
  L.counts_off = off;
  off = align_up(off + sizeof(uint32_t) * img->batch, 256);
  L.edges_off = off;
  off = align_up(off + sizeof(uint32_t) * static_cast<size_t>(L.edge_stride) * img->batch, 256);
  L.acc_off = off;
  if (acc_ws) off = align_up(off + acc_bytes, 256);
  L.hint_off = off;
  off = align_up(off + hint_bytes(img->batch, n_theta, 2 * d + 1), 256);
  L.peaks_off = off;
  off = align_up(off + peaks_workspace_bytes(img->batch, n_theta, 2 * d + 1, k), 256);
  L.total = off;
  return L;
}

}  // namespace ld


// An NVTX range over one ABI call (nsys / ncu --nvtx timelines name the
// library's stages; inert without a tool attached).
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

using namespace ld;

extern "C" {

int32_t ld_rho_offset(int32_t width, int32_t height) { return rho_offset(width, height); }

const char *ld_status_string(int status) {
  switch (status) {
    case LD_OK: return "LD_OK";
    case LD_ERR_INVALID_ARG: return "LD_ERR_INVALID_ARG";
    case LD_ERR_RANGE: return "LD_ERR_RANGE";
    case LD_ERR_WORKSPACE: return "LD_ERR_WORKSPACE";
    case LD_ERR_UNSUPPORTED: return "LD_ERR_UNSUPPORTED";
    case LD_ERR_CUDA: return "LD_ERR_CUDA";
    default: return "LD_ERR_UNKNOWN";
  }
}

const char *ld_last_error_detail(void) { return g_err; }

int32_t ld_last_launch_count(void) { return g_launches; }

int32_t ld_device_sm_count(void) {
  DevInfo d;
  device_info(&d);
  return d.sm_count;
}

int64_t ld_device_l2_bytes(void) {
  DevInfo d;
  device_info(&d);
  return d.l2;
}

int ld_sobel_binarize_ex(const uint8_t *gray, const ld_image *img, int32_t threshold,
                         uint32_t flags, uint8_t *binary, uint32_t *edge_xy,
                         int64_t edge_stride, uint32_t *edge_count, void *stream) {
  NvtxRange nvtx_range_("ld_sobel_binarize_ex");
  g_launches = 0;
  int rc = check_image(gray, img);
  if (rc) return rc;
  if (flags & ~static_cast<uint32_t>(LD_FLAG_ZERO_PAD | LD_FLAG_CLAMP_255))
    return fail(LD_ERR_INVALID_ARG, "unknown flag bits 0x%x", flags);
  if (!edge_count) return fail(LD_ERR_INVALID_ARG, "edge_count is NULL");
  if (edge_xy && edge_stride < max_edges_per_frame(img, flags))
    return fail(LD_ERR_INVALID_ARG, "edge_stride %lld < %lld possible edges per frame",
                static_cast<long long>(edge_stride),
                static_cast<long long>(max_edges_per_frame(img, flags)));
  if (binary && !aligned(binary, 16)) return fail(LD_ERR_INVALID_ARG, "binary must be 16-byte aligned");
  return sobel_impl(gray, img, threshold, flags, binary, edge_xy, edge_stride, edge_count,
                    static_cast<cudaStream_t>(stream));
}

int ld_sobel_binarize(const uint8_t *gray, const ld_image *img, int32_t threshold,
                      uint8_t *binary, uint32_t *edge_xy, int64_t edge_stride,
                      uint32_t *edge_count, void *stream) {
  return ld_sobel_binarize_ex(gray, img, threshold, 0u, binary, edge_xy, edge_stride, edge_count,
                              stream);
}

static int check_vote_args(const uint32_t *edge_xy, const uint32_t *edge_count, const uint32_t *acc,
                           int64_t edge_stride, int32_t batch, int32_t width, int32_t height) {
  if (!edge_xy || !edge_count || !acc) return fail(LD_ERR_INVALID_ARG, "NULL device pointer");
  if (batch < 1) return fail(LD_ERR_INVALID_ARG, "batch must be >= 1");
  if (width < 1 || height < 1 || width > LD_MAX_DIM || height > LD_MAX_DIM)
    return fail(LD_ERR_INVALID_ARG, "width/height outside [1, %d]", LD_MAX_DIM);
  if (!aligned(edge_xy, 16) || edge_stride < 0 || edge_stride % 4 != 0)
    return fail(LD_ERR_INVALID_ARG, "edge_xy must be 16-byte aligned and edge_stride a multiple of 4");
  return LD_OK;
}

int ld_hough_accumulate_opt(const uint32_t *edge_xy, const uint32_t *edge_count,
                            int64_t edge_stride, int32_t batch, int32_t width, int32_t height,
                            int32_t n_theta, const int32_t *cos_q15, const int32_t *sin_q15,
                            uint32_t flags, uint32_t *acc, void *hint, size_t hint_bytes_,
                            void *stream) {
  NvtxRange nvtx_range_("ld_hough_accumulate_opt");
  g_launches = 0;
  int rc = check_vote_args(edge_xy, edge_count, acc, edge_stride, batch, width, height);
  if (rc) return rc;
  if (flags & ~static_cast<uint32_t>(LD_VOTE_PLAIN | LD_VOTE_NO_CLUSTER))
    return fail(LD_ERR_INVALID_ARG, "unknown flag bits 0x%x", flags);
  if (n_theta < 1 || n_theta > LD_MAX_THETA)
    return fail(LD_ERR_INVALID_ARG, "n_theta %d outside [1, %d]", n_theta, LD_MAX_THETA);
  if (hint) {
    const size_t need = hint_bytes(batch, n_theta, 2 * rho_offset(width, height) + 1);
    if (!aligned(hint, 16) || hint_bytes_ < need)
      return fail(LD_ERR_WORKSPACE, "hint needs %zu bytes, 16-byte aligned", need);
  }
  return hough_impl(edge_xy, edge_count, edge_stride, batch, width, height, n_theta, cos_q15,
                    sin_q15, acc, static_cast<cudaStream_t>(stream), hint, flags);
}

int ld_hough_accumulate(const uint32_t *edge_xy, const uint32_t *edge_count, int64_t edge_stride,
                        int32_t batch, int32_t width, int32_t height, int32_t n_theta,
                        const int32_t *cos_q15, const int32_t *sin_q15, uint32_t *acc,
                        void *stream) {
  return ld_hough_accumulate_opt(edge_xy, edge_count, edge_stride, batch, width, height, n_theta,
                                 cos_q15, sin_q15, 0u, acc, nullptr, 0, stream);
}

int ld_hough_accumulate_f64(const uint32_t *edge_xy, const uint32_t *edge_count,
                            int64_t edge_stride, int32_t batch, int32_t width, int32_t height,
                            int32_t n_theta, const double *cos_f64, const double *sin_f64,
                            uint32_t *acc, void *stream) {
  NvtxRange nvtx_range_("ld_hough_accumulate_f64");
  g_launches = 0;
  const int rc0 = check_vote_args(edge_xy, edge_count, acc, edge_stride, batch, width, height);
  if (rc0) return rc0;
  if (n_theta < 1 || n_theta > LD_MAX_THETA_F64)
    return fail(LD_ERR_INVALID_ARG, "n_theta %d outside [1, %d]", n_theta, LD_MAX_THETA_F64);
  if (!cos_f64 || !sin_f64) return fail(LD_ERR_INVALID_ARG, "trig table pointer is NULL");
  const int32_t d = rho_offset(width, height);
  const int64_t n_rho = 2 * static_cast<int64_t>(d) + 1;
  const double xs[2] = {0.0, static_cast<double>(width - 1)};
  const double ys[2] = {0.0, static_cast<double>(height - 1)};
  for (int t = 0; t < n_theta; ++t) {
    const double c = cos_f64[t], s = sin_f64[t];
    if (!(c >= -1.0 && c <= 1.0 && s >= -1.0 && s <= 1.0))
      return fail(LD_ERR_RANGE, "trig entry %d (%g, %g) is not finite in [-1, 1]", t, c, s);
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        volatile double px = xs[a] * c;  // rounded on its own (no contraction)
        volatile double py = ys[b] * s;
        const double r = px + py;
        const int64_t rho = static_cast<int64_t>(floor(r + 0.5)) + d;
        if (rho < 0 || rho >= n_rho)
          return fail(LD_ERR_RANGE, "theta bin %d sends a corner to rho bin %lld", t,
                      static_cast<long long>(rho));
      }
  }
  DevInfo dev;
  int rc = device_info(&dev);
  if (rc) return rc;
  int ctas = 1, rpb = 0, n_bands = 0;
  size_t smem = 0;
  if (!hough_plan(n_theta, static_cast<int>(n_rho), static_cast<size_t>(dev.smem_optin), &ctas,
                  &rpb, &n_bands, &smem))
    return fail(LD_ERR_UNSUPPORTED, "one accumulator row (%lld bins) exceeds shared memory",
                static_cast<long long>(n_rho));
  static thread_local TrigTableF64 trig;
  memcpy(trig.c, cos_f64, sizeof(double) * n_theta);
  memcpy(trig.s, sin_f64, sizeof(double) * n_theta);
  HoughParams p;
  memset(&p, 0, sizeof(p));
  p.edges = edge_xy;
  p.counts = edge_count;
  p.edge_stride = edge_stride;
  p.batch = batch;
  p.n_theta = n_theta;
  p.n_rho = static_cast<int32_t>(n_rho);
  p.rows_per_band = rpb;
  p.n_bands = n_bands;
  p.acc = acc;
  cudaError_t e = launch_hough_f64(p, trig, ctas, smem, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "hough_vote_f64_kernel launch");
  return LD_OK;
}

size_t ld_hough_hint_bytes(int32_t batch, int32_t width, int32_t height, int32_t n_theta) {
  if (batch < 1 || width < 1 || height < 1 || n_theta < 1) return 0;
  return hint_bytes(batch, n_theta, 2 * rho_offset(width, height) + 1);
}

int ld_hough_accumulate_hint(const uint32_t *edge_xy, const uint32_t *edge_count,
                             int64_t edge_stride, int32_t batch, int32_t width, int32_t height,
                             int32_t n_theta, const int32_t *cos_q15, const int32_t *sin_q15,
                             uint32_t *acc, void *hint, size_t hint_bytes_, void *stream) {
  NvtxRange nvtx_range_("ld_hough_accumulate_hint");
  if (!hint) {
    g_launches = 0;
    return fail(LD_ERR_INVALID_ARG, "NULL hint");
  }
  return ld_hough_accumulate_opt(edge_xy, edge_count, edge_stride, batch, width, height, n_theta,
                                 cos_q15, sin_q15, 0u, acc, hint, hint_bytes_, stream);
}

size_t ld_hough_peaks_workspace_bytes(int32_t batch, int32_t n_theta, int32_t n_rho, int32_t k) {
  if (batch < 1 || n_theta < 1 || n_rho < 1 || k < 1) return 0;
  return peaks_workspace_bytes(batch, n_theta, n_rho, k);
}

int ld_hough_peaks_opt(const uint32_t *acc, int32_t batch, int32_t n_theta, int32_t n_rho,
                       int32_t half_theta, int32_t half_rho, uint32_t min_votes, int32_t k,
                       int32_t cand_row_begin, int32_t cand_row_end, int32_t theta_offset,
                       const void *hint, size_t hint_bytes_, uint32_t flags, ld_peak *peaks,
                       int32_t *n_peaks, void *workspace, size_t workspace_bytes,
                       void *stream) {
  NvtxRange nvtx_range_("ld_hough_peaks_opt");
  g_launches = 0;
  int rc = check_peaks_args(acc, batch, n_theta, n_rho, half_theta, half_rho, k, peaks, n_peaks);
  if (rc) return rc;
  if (flags & ~static_cast<uint32_t>(LD_PEAKS_DENSE | LD_PEAKS_FORCE_STREAM | LD_PEAKS_FORCE_TILE |
                                     LD_PEAKS_FORCE_BAND))
    return fail(LD_ERR_INVALID_ARG, "unknown flag bits 0x%x", flags);
  if (cand_row_begin < 0 || cand_row_end < cand_row_begin || cand_row_end > n_theta)
    return fail(LD_ERR_INVALID_ARG, "candidate rows [%d, %d) outside [0, %d]", cand_row_begin,
                cand_row_end, n_theta);
  if (theta_offset < 0 ||
      (static_cast<int64_t>(theta_offset) + n_theta) * n_rho >= (1ll << 32) - 1)
    return fail(LD_ERR_INVALID_ARG, "theta_offset %d: global cell index exceeds 32 bits",
                theta_offset);
  if (hint && (!aligned(hint, 16) || hint_bytes_ < hint_bytes(batch, n_theta, n_rho)))
    return fail(LD_ERR_WORKSPACE, "hint needs %zu bytes, 16-byte aligned",
                hint_bytes(batch, n_theta, n_rho));
  DevInfo dev;
  if ((rc = device_info(&dev))) return rc;
  if (!workspace || !aligned(workspace, 16) ||
      workspace_bytes < peaks_workspace_bytes(batch, n_theta, n_rho, k))
    return fail(LD_ERR_WORKSPACE, "workspace needs %zu bytes, 16-byte aligned",
                peaks_workspace_bytes(batch, n_theta, n_rho, k));
  return peaks_impl(acc, batch, n_theta, n_rho, half_theta, half_rho, min_votes, k, peaks,
                    n_peaks, workspace, workspace_bytes, static_cast<cudaStream_t>(stream),
                    cand_row_begin, cand_row_end, theta_offset, hint, flags);
}

int ld_hough_peaks_ex(const uint32_t *acc, int32_t batch, int32_t n_theta, int32_t n_rho,
                      int32_t half_theta, int32_t half_rho, uint32_t min_votes, int32_t k,
                      int32_t cand_row_begin, int32_t cand_row_end, int32_t theta_offset,
                      ld_peak *peaks, int32_t *n_peaks, void *workspace,
                      size_t workspace_bytes, void *stream) {
  return ld_hough_peaks_opt(acc, batch, n_theta, n_rho, half_theta, half_rho, min_votes, k,
                            cand_row_begin, cand_row_end, theta_offset, nullptr, 0, 0u, peaks,
                            n_peaks, workspace, workspace_bytes, stream);
}

int ld_hough_hint_from_acc(const uint32_t *acc, int32_t batch, int32_t n_theta, int32_t n_rho,
                           int32_t cand_row_begin, int32_t cand_row_end, void *hint,
                           size_t hint_bytes_, void *stream) {
  NvtxRange nvtx_range_("ld_hough_hint_from_acc");
  g_launches = 0;
  if (!acc || !hint) return fail(LD_ERR_INVALID_ARG, "NULL acc/hint");
  if (batch < 1 || n_theta < 1 || n_theta > LD_MAX_THETA || n_rho < 1)
    return fail(LD_ERR_INVALID_ARG, "bad accumulator shape [%d][%d][%d]", batch, n_theta, n_rho);
  if (static_cast<int64_t>(n_theta) * n_rho >= (1ll << 31))
    return fail(LD_ERR_INVALID_ARG, "a frame of %d x %d counters exceeds 2^31", n_theta, n_rho);
  if (cand_row_begin < 0 || cand_row_end < cand_row_begin || cand_row_end > n_theta)
    return fail(LD_ERR_INVALID_ARG, "candidate rows [%d, %d) outside [0, %d]", cand_row_begin,
                cand_row_end, n_theta);
  if (!aligned(acc, 4)) return fail(LD_ERR_INVALID_ARG, "acc not 4-byte aligned");
  if (!aligned(hint, 16) || hint_bytes_ < hint_bytes(batch, n_theta, n_rho))
    return fail(LD_ERR_WORKSPACE, "hint needs %zu bytes, 16-byte aligned",
                hint_bytes(batch, n_theta, n_rho));
  DevInfo dev;
  int rc = device_info(&dev);
  if (rc) return rc;
  char *hb = static_cast<char *>(hint);
  const cudaError_t e = launch_hint_from_acc(
      acc, batch, n_theta, n_rho, cand_row_begin, cand_row_end, reinterpret_cast<uint32_t *>(hb),
      reinterpret_cast<unsigned long long *>(hb + HINT_HDR_BYTES),
      reinterpret_cast<uint32_t *>(hb + HINT_HDR_BYTES + hint_keys_bytes(batch, n_theta)),
      static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "hint_from_acc_kernel launch");
  return LD_OK;
}

int ld_hough_peaks_hinted(const uint32_t *acc, int32_t batch, int32_t n_theta, int32_t n_rho,
                          int32_t half_theta, int32_t half_rho, uint32_t min_votes, int32_t k,
                          const void *hint, size_t hint_bytes_, ld_peak *peaks, int32_t *n_peaks,
                          void *workspace, size_t workspace_bytes, void *stream) {
  if (!hint) {
    g_launches = 0;
    const int rc = check_peaks_args(acc, batch, n_theta, n_rho, half_theta, half_rho, k, peaks,
                                    n_peaks);
    if (rc) return rc;
    return fail(LD_ERR_WORKSPACE, "hint needs %zu bytes, 16-byte aligned",
                hint_bytes(batch, n_theta, n_rho));
  }
  return ld_hough_peaks_opt(acc, batch, n_theta, n_rho, half_theta, half_rho, min_votes, k, 0,
                            n_theta, 0, hint, hint_bytes_, 0u, peaks, n_peaks, workspace,
                            workspace_bytes, stream);
}

int ld_hough_peaks(const uint32_t *acc, int32_t batch, int32_t n_theta, int32_t n_rho,
                   int32_t half_theta, int32_t half_rho, uint32_t min_votes, int32_t k,
                   ld_peak *peaks, int32_t *n_peaks, void *workspace, size_t workspace_bytes,
                   void *stream) {
  return ld_hough_peaks_opt(acc, batch, n_theta, n_rho, half_theta, half_rho, min_votes, k, 0,
                            n_theta, 0, nullptr, 0, 0u, peaks, n_peaks, workspace,
                            workspace_bytes, stream);
}

size_t ld_detect_workspace_bytes(const ld_image *img, int32_t n_theta, int32_t k,
                                 int32_t acc_in_workspace) {
  if (!img || img->batch < 1 || img->width < 1 || img->height < 1 || n_theta < 1 || k < 1) return 0;
  ld_image whole = *img;
  whole.row_begin = 0;
  whole.row_end = img->height;
  return detect_layout(&whole, n_theta, k, acc_in_workspace != 0).total;
}

// ---------------------------------------------------------------------------
// Lanes module (NEXT 3)
// ---------------------------------------------------------------------------
static size_t nms_layout(int32_t batch, int32_t n_theta, int32_t n_rho, int64_t *words,
                         size_t *bitmap_off) {
  *words = (static_cast<int64_t>(n_theta) * n_rho + 31) / 32;
  *bitmap_off = align_up(sizeof(NmsState) * static_cast<size_t>(batch), 256);
  return *bitmap_off + sizeof(uint32_t) * static_cast<size_t>(*words) * batch;
}

size_t ld_hough_peaks_nms_workspace_bytes(int32_t batch, int32_t n_theta, int32_t n_rho) {
  if (batch < 1 || n_theta < 1 || n_rho < 1) return 0;
  int64_t w;
  size_t off;
  return nms_layout(batch, n_theta, n_rho, &w, &off);
}

int ld_hough_peaks_nms(const uint32_t *acc, int32_t batch, int32_t n_theta, int32_t n_rho,
                       int32_t half_theta, int32_t half_rho, uint32_t min_votes,
                       uint32_t ratio_num, uint32_t ratio_den, int32_t k, ld_peak *peaks,
                       int32_t *n_peaks, void *workspace, size_t workspace_bytes,
                       void *stream) {
  NvtxRange nvtx_range_("ld_hough_peaks_nms");
  g_launches = 0;
  int rc = check_peaks_args(acc, batch, n_theta, n_rho, half_theta, half_rho, k, peaks, n_peaks);
  if (rc) return rc;
  if (ratio_den < 1) return fail(LD_ERR_INVALID_ARG, "ratio_den must be >= 1");
  int64_t words;
  size_t off;
  const size_t need = nms_layout(batch, n_theta, n_rho, &words, &off);
  if (!workspace || !aligned(workspace, 16) || workspace_bytes < need)
    return fail(LD_ERR_WORKSPACE, "workspace needs %zu bytes, 16-byte aligned", need);
  DevInfo dev;
  if ((rc = device_info(&dev))) return rc;
  NmsParams p;
  p.acc = acc;
  p.batch = batch;
  p.n_theta = n_theta;
  p.n_rho = n_rho;
  p.half_theta = half_theta;
  p.half_rho = half_rho;
  p.k = k;
  p.floor_votes = min_votes > 1 ? min_votes : 1u;
  p.ratio_num = ratio_num;
  p.ratio_den = ratio_den;
  p.state = static_cast<NmsState *>(workspace);
  p.bitmap = reinterpret_cast<uint32_t *>(static_cast<char *>(workspace) + off);
  p.bitmap_words = words;
  p.peaks = peaks;
  p.n_peaks = n_peaks;
  cudaError_t e = launch_nms(p, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "NMS kernels launch");
  return LD_OK;
}

static int lanes_common(const ld_peak *peaks, const int32_t *n_peaks, int32_t batch, int32_t k,
                        int32_t width, int32_t height, int32_t n_theta, const int32_t *c,
                        const int32_t *s, LanesParams *p, TrigTable *trig) {
  if (!peaks || !n_peaks) return fail(LD_ERR_INVALID_ARG, "NULL peaks/n_peaks");
  if (batch < 1 || k < 1 || k > LD_MAX_K) return fail(LD_ERR_INVALID_ARG, "bad batch/k");
  if (width < 1 || height < 1 || width > LD_MAX_DIM || height > LD_MAX_DIM)
    return fail(LD_ERR_INVALID_ARG, "width/height outside [1, %d]", LD_MAX_DIM);
  if (n_theta < 1 || n_theta > LD_MAX_THETA || !c || !s)
    return fail(LD_ERR_INVALID_ARG, "bad trig table");
  for (int t = 0; t < n_theta; ++t)
    if (c[t] < -32768 || c[t] > 32768 || s[t] < -32768 || s[t] > 32768)
      return fail(LD_ERR_RANGE, "trig entry %d (%d, %d) exceeds |32768|", t, c[t], s[t]);
  DevInfo dev;
  int rc = device_info(&dev);
  if (rc) return rc;
  memset(p, 0, sizeof(*p));
  p->peaks = peaks;
  p->n_peaks = n_peaks;
  p->batch = batch;
  p->k = k;
  p->width = width;
  p->height = height;
  p->n_theta = n_theta;
  p->rho_offset = rho_offset(width, height);
  memcpy(trig->c, c, sizeof(int32_t) * n_theta);
  memcpy(trig->s, s, sizeof(int32_t) * n_theta);
  return LD_OK;
}

int ld_peak_lines(const ld_peak *peaks, const int32_t *n_peaks, int32_t batch, int32_t k,
                  int32_t width, int32_t height, int32_t n_theta, const int32_t *cos_q15,
                  const int32_t *sin_q15, ld_segment *lines, int32_t *hit, void *stream) {
  NvtxRange nvtx_range_("ld_peak_lines");
  g_launches = 0;
  static thread_local TrigTable trig;
  LanesParams p;
  int rc = lanes_common(peaks, n_peaks, batch, k, width, height, n_theta, cos_q15, sin_q15, &p,
                        &trig);
  if (rc) return rc;
  if (!lines || !hit) return fail(LD_ERR_INVALID_ARG, "NULL lines/hit");
  p.lines = lines;
  p.hit = hit;
  cudaError_t e = launch_peak_lines(p, trig, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "peak_lines_kernel launch");
  return LD_OK;
}

int ld_extract_segments(const uint8_t *binary, const ld_image *img, const ld_peak *peaks,
                        const int32_t *n_peaks, int32_t k, int32_t n_theta,
                        const int32_t *cos_q15, const int32_t *sin_q15, int32_t fill_gap,
                        int32_t min_len, int32_t max_segments, ld_segment *segments,
                        int32_t *n_segments, void *stream) {
  NvtxRange nvtx_range_("ld_extract_segments");
  g_launches = 0;
  if (!img || !binary) return fail(LD_ERR_INVALID_ARG, "NULL binary/img");
  if (img->pitch < img->width || img->batch < 1 ||
      (img->batch > 1 && img->frame_stride < static_cast<int64_t>(img->height) * img->pitch))
    return fail(LD_ERR_INVALID_ARG, "binary geometry: pitch >= width, frame_stride >= height*pitch");
  if (fill_gap < 0 || min_len < 0 || max_segments < 1)
    return fail(LD_ERR_INVALID_ARG, "fill_gap, min_len >= 0 and max_segments >= 1");
  if (!segments || !n_segments) return fail(LD_ERR_INVALID_ARG, "NULL segments/n_segments");
  static thread_local TrigTable trig;
  LanesParams p;
  int rc = lanes_common(peaks, n_peaks, img->batch, k, img->width, img->height, n_theta, cos_q15,
                        sin_q15, &p, &trig);
  if (rc) return rc;
  p.binary = binary;
  p.bin_pitch = img->pitch;
  p.bin_frame_stride = img->batch > 1 ? img->frame_stride : static_cast<int64_t>(img->height) * img->pitch;
  p.fill_gap = fill_gap;
  p.min_len = min_len;
  p.max_segs = max_segments;
  p.segs = segments;
  p.n_segs = n_segments;
  cudaError_t e = launch_extract_segments(p, trig, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "extract_segments_kernel launch");
  return LD_OK;
}

int ld_detect_batch_ex(const uint8_t *gray, const ld_image *img, int32_t threshold,
                       uint32_t flags, int32_t n_theta, const int32_t *cos_q15,
                       const int32_t *sin_q15, int32_t half_theta, int32_t half_rho,
                       uint32_t min_votes, int32_t k, ld_peak *peaks, int32_t *n_peaks,
                       uint32_t *edge_count, uint32_t *acc, void *workspace,
                       size_t workspace_bytes, void *stream) {
  NvtxRange nvtx_range_("ld_detect_batch_ex");
  g_launches = 0;
  int rc = check_image(gray, img);
  if (rc) return rc;
  if (flags & ~static_cast<uint32_t>(LD_FLAG_ZERO_PAD | LD_FLAG_CLAMP_255))
    return fail(LD_ERR_INVALID_ARG, "unknown flag bits 0x%x", flags);
  if (img->row_begin != 0 || img->row_end != img->height)
    return fail(LD_ERR_INVALID_ARG, "ld_detect_batch takes whole frames (rows [0, height))");
  const int32_t d = rho_offset(img->width, img->height);
  const int32_t n_rho = 2 * d + 1;
  if ((rc = check_trig(n_theta, cos_q15, sin_q15, img->width, img->height, d))) return rc;
  if ((rc = check_peaks_args(acc ? acc : reinterpret_cast<uint32_t *>(16), img->batch, n_theta,
                             n_rho, half_theta, half_rho, k, peaks, n_peaks)))
    return rc;
  const DetectLayout L = detect_layout(img, n_theta, k, acc == nullptr);
  if (!workspace || !aligned(workspace, 256) || workspace_bytes < L.total)
    return fail(LD_ERR_WORKSPACE, "workspace needs %zu bytes, 256-byte aligned", L.total);
  if (acc && !aligned(acc, 16)) return fail(LD_ERR_INVALID_ARG, "acc must be 16-byte aligned");
  char *ws = static_cast<char *>(workspace);
  uint32_t *counts = reinterpret_cast<uint32_t *>(ws + L.counts_off);
  uint32_t *edges = reinterpret_cast<uint32_t *>(ws + L.edges_off);
  uint32_t *A = acc ? acc : reinterpret_cast<uint32_t *>(ws + L.acc_off);
  void *pws = ws + L.peaks_off;
  void *hint = ws + L.hint_off;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((rc = sobel_impl(gray, img, threshold, flags, nullptr, edges, L.edge_stride, counts, s)))
    return rc;
  if ((rc = hough_impl(edges, counts, L.edge_stride, img->batch, img->width, img->height, n_theta,
                       cos_q15, sin_q15, A, s, hint)))
    return rc;
  if ((rc = peaks_impl(A, img->batch, n_theta, n_rho, half_theta, half_rho, min_votes, k, peaks,
                       n_peaks, pws, workspace_bytes - L.peaks_off, s, 0, -1, 0, hint)))
    return rc;
  if (edge_count) {
    cudaError_t e = cudaMemcpyAsync(edge_count, counts, sizeof(uint32_t) * img->batch,
                                    cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(edge_count)");
  }
  return LD_OK;
}

int ld_detect_batch(const uint8_t *gray, const ld_image *img, int32_t threshold, int32_t n_theta,
                    const int32_t *cos_q15, const int32_t *sin_q15, int32_t half_theta,
                    int32_t half_rho, uint32_t min_votes, int32_t k, ld_peak *peaks,
                    int32_t *n_peaks, uint32_t *edge_count, uint32_t *acc, void *workspace,
                    size_t workspace_bytes, void *stream) {
  return ld_detect_batch_ex(gray, img, threshold, 0u, n_theta, cos_q15, sin_q15, half_theta,
                            half_rho, min_votes, k, peaks, n_peaks, edge_count, acc, workspace,
                            workspace_bytes, stream);
}

// ---------------------------------------------------------------------------
// Host-buffer path: chunked, double-buffered H2D overlapped with the kernels.
// Device workspace layout: [2][chunk][frame_stride] gray staging, then for each
// of the 2 slots {peaks[chunk][k], n_peaks[chunk], counts[chunk]}, then one
// ld_detect_batch workspace sized for `chunk` frames (acc in workspace).
// ---------------------------------------------------------------------------
struct HostLayout {
  size_t gray_off[2], peaks_off[2], npk_off[2], cnt_off[2], det_off, det_bytes, total;
  int64_t fstride;
};

static HostLayout host_layout(const ld_image *img, int32_t n_theta, int32_t k, int32_t chunk) {
  HostLayout L;
  L.fstride = img->batch > 1 ? img->frame_stride : static_cast<int64_t>(img->height) * img->pitch;
  size_t off = 0;
  for (int i = 0; i < 2; ++i) {
    L.gray_off[i] = off;
    off = align_up(off + static_cast<size_t>(L.fstride) * chunk, 256);
  }
  for (int i = 0; i < 2; ++i) {
    L.peaks_off[i] = off;
    off = align_up(off + sizeof(ld_peak) * static_cast<size_t>(k) * chunk, 256);
    L.npk_off[i] = off;
    off = align_up(off + sizeof(int32_t) * chunk, 256);
    L.cnt_off[i] = off;
    off = align_up(off + sizeof(uint32_t) * chunk, 256);
  }
  ld_image ci = *img;
  ci.batch = chunk;
  ci.row_begin = 0;
  ci.row_end = img->height;
  L.det_off = off;
  L.det_bytes = detect_layout(&ci, n_theta, k, true).total;
  L.total = off + L.det_bytes;
  return L;
}

// The host path's copy stream and its 4 events, created once per (host
// thread, device) and kept for the thread's lifetime (a thread-local cache:
// no shared mutable state, no per-call creation).  Each call synchronises
// both streams before returning, so reuse is safe.
struct HostStreams {
  bool ok = false;
  cudaStream_t copy = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
};

static int host_streams(HostStreams **out) {
  static thread_local HostStreams per_dev[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  HostStreams &h = per_dev[dev & 63];
  if (!h.ok) {
    e = cudaStreamCreateWithFlags(&h.copy, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
      e = cudaEventCreateWithFlags(&h.copied[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h.done[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) return cuda_fail(e, "stream/event creation");
    h.ok = true;
  }
  *out = &h;
  return LD_OK;
}

size_t ld_detect_host_workspace_bytes(const ld_image *img, int32_t n_theta, int32_t k,
                                      int32_t chunk_frames) {
  if (!img || img->batch < 1 || chunk_frames < 1 || n_theta < 1 || k < 1) return 0;
  const int32_t chunk = chunk_frames < img->batch ? chunk_frames : img->batch;
  return host_layout(img, n_theta, k, chunk).total;
}

int ld_detect_batch_host(const uint8_t *gray_host, const ld_image *img, int32_t threshold,
                         int32_t n_theta, const int32_t *cos_q15, const int32_t *sin_q15,
                         int32_t half_theta, int32_t half_rho, uint32_t min_votes, int32_t k,
                         ld_peak *peaks_host, int32_t *n_peaks_host, uint32_t *edge_count_host,
                         int32_t chunk_frames, void *workspace, size_t workspace_bytes,
                         void *stream) {
  NvtxRange nvtx_range_("ld_detect_batch_host");
  if (!gray_host || !img || !peaks_host || !n_peaks_host)
    return fail(LD_ERR_INVALID_ARG, "NULL host pointer");
  if (chunk_frames < 1) return fail(LD_ERR_INVALID_ARG, "chunk_frames must be >= 1");
  if (img->row_begin != 0 || img->row_end != img->height)
    return fail(LD_ERR_INVALID_ARG, "ld_detect_batch_host takes whole frames");
  const int32_t chunk = chunk_frames < img->batch ? chunk_frames : img->batch;
  const HostLayout L = host_layout(img, n_theta, k, chunk);
  if (!workspace || !aligned(workspace, 256) || workspace_bytes < L.total)
    return fail(LD_ERR_WORKSPACE, "workspace needs %zu bytes, 256-byte aligned", L.total);
  int launches = 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HostStreams *hs = nullptr;
  int rc = host_streams(&hs);
  cudaError_t e = cudaSuccess;
  cudaStream_t cs = hs ? hs->copy : nullptr;
  cudaEvent_t *copied = hs ? hs->copied : nullptr, *done = hs ? hs->done : nullptr;
  char *ws = static_cast<char *>(workspace);
  const int n_chunks = (img->batch + chunk - 1) / chunk;
  // the copy stream must not start before earlier work on `stream` that may use the workspace
  if (rc == LD_OK) {
    e = cudaEventRecord(done[1], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, done[1], 0);
    if (e != cudaSuccess) rc = cuda_fail(e, "initial ordering");
  }
  for (int ci = 0; ci < n_chunks && rc == LD_OK; ++ci) {
    const int slot = ci & 1;
    const int f0 = ci * chunk;
    const int nf = img->batch - f0 < chunk ? img->batch - f0 : chunk;
    uint8_t *dgray = reinterpret_cast<uint8_t *>(ws + L.gray_off[slot]);
    if (ci >= 2) {  // slot reuse: wait for the kernels of chunk ci-2
      e = cudaStreamWaitEvent(cs, done[slot], 0);
      if (e != cudaSuccess) { rc = cuda_fail(e, "cudaStreamWaitEvent"); break; }
    }
    e = cudaMemcpyAsync(dgray, gray_host + static_cast<int64_t>(f0) * L.fstride,
                        static_cast<size_t>(L.fstride) * nf, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess) e = cudaEventRecord(copied[slot], cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, copied[slot], 0);
    if (e != cudaSuccess) { rc = cuda_fail(e, "H2D copy"); break; }
    ld_image ci_img = *img;
    ci_img.batch = nf;
    ci_img.frame_stride = L.fstride;
    ld_peak *dpk = reinterpret_cast<ld_peak *>(ws + L.peaks_off[slot]);
    int32_t *dnp = reinterpret_cast<int32_t *>(ws + L.npk_off[slot]);
    uint32_t *dcnt = reinterpret_cast<uint32_t *>(ws + L.cnt_off[slot]);
    rc = ld_detect_batch(dgray, &ci_img, threshold, n_theta, cos_q15, sin_q15, half_theta,
                         half_rho, min_votes, k, dpk, dnp, dcnt, nullptr, ws + L.det_off,
                         L.det_bytes, s);
    launches += g_launches;
    if (rc) break;
    e = cudaEventRecord(done[slot], s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(peaks_host + static_cast<int64_t>(f0) * k, dpk,
                          sizeof(ld_peak) * static_cast<size_t>(k) * nf, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(n_peaks_host + f0, dnp, sizeof(int32_t) * nf, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && edge_count_host)
      e = cudaMemcpyAsync(edge_count_host + f0, dcnt, sizeof(uint32_t) * nf,
                          cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) { rc = cuda_fail(e, "D2H copy"); break; }
  }
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess && rc == LD_OK) rc = cuda_fail(e, "cudaStreamSynchronize");
  if (cs) cudaStreamSynchronize(cs);
  g_launches = launches;
  return rc;
}

int64_t ld_edge_bitmask_words(int32_t width, int32_t rows) {
  if (width < 1 || rows < 1) return 0;
  return static_cast<int64_t>(rows) * ((width + 31) / 32);
}

int ld_edges_to_bitmask(const uint32_t *edge_xy, const uint32_t *edge_count, int32_t width,
                        int32_t row_begin, int32_t rows, uint32_t *bits, void *stream) {
  NvtxRange nvtx_range_("ld_edges_to_bitmask");
  g_launches = 0;
  if (!edge_xy || !edge_count || !bits) return fail(LD_ERR_INVALID_ARG, "NULL device pointer");
  if (width < 1 || width > LD_MAX_DIM || rows < 1 || row_begin < 0 ||
      row_begin + rows > LD_MAX_DIM)
    return fail(LD_ERR_INVALID_ARG, "bad band: width %d, rows [%d, %d)", width, row_begin,
                row_begin + rows);
  if (!aligned(bits, 16)) return fail(LD_ERR_INVALID_ARG, "bits must be 16-byte aligned");
  DevInfo dev;
  int rc = device_info(&dev);
  if (rc) return rc;
  cudaError_t e = launch_edges_to_bitmask(edge_xy, edge_count, width, row_begin, rows, bits,
                                          dev.sm_count, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "edges_to_bitmask_kernel launch");
  return LD_OK;
}

int ld_bitmask_to_edges(const uint32_t *bits, int32_t width, int32_t n_blocks,
                        const int32_t *block_row_begin, const int32_t *block_rows,
                        int32_t block_stride_rows, uint32_t *edge_xy, int64_t edge_capacity,
                        uint32_t *edge_count, void *stream) {
  NvtxRange nvtx_range_("ld_bitmask_to_edges");
  g_launches = 0;
  if (!bits || !edge_xy || !edge_count) return fail(LD_ERR_INVALID_ARG, "NULL device pointer");
  if (!block_row_begin || !block_rows) return fail(LD_ERR_INVALID_ARG, "NULL block table");
  if (width < 1 || width > LD_MAX_DIM || n_blocks < 1 || n_blocks > LD_MAX_BLOCKS ||
      block_stride_rows < 1 || edge_capacity < 0)
    return fail(LD_ERR_INVALID_ARG, "bad bitmap geometry");
  for (int b = 0; b < n_blocks; ++b)
    if (block_rows[b] < 0 || block_rows[b] > block_stride_rows || block_row_begin[b] < 0 ||
        block_row_begin[b] + block_rows[b] > LD_MAX_DIM)
      return fail(LD_ERR_INVALID_ARG, "block %d: rows [%d, +%d) invalid", b, block_row_begin[b],
                  block_rows[b]);
  DevInfo dev;
  int rc = device_info(&dev);
  if (rc) return rc;
  cudaError_t e = launch_bitmask_to_edges(bits, width, n_blocks, block_row_begin, block_rows,
                                          block_stride_rows, edge_xy, edge_capacity, edge_count,
                                          static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "bitmask_to_edges_kernel launch");
  return LD_OK;
}

int ld_merge_peak_lists(const ld_peak *peaks, const int32_t *n_peaks, int32_t n_lists,
                        int32_t k, int32_t n_rho, ld_peak *out, int32_t *n_out, void *stream) {
  NvtxRange nvtx_range_("ld_merge_peak_lists");
  g_launches = 0;
  if (!peaks || !n_peaks || !out || !n_out) return fail(LD_ERR_INVALID_ARG, "NULL device pointer");
  if (n_lists < 1 || k < 1 || k > LD_MAX_K || n_rho < 1 ||
      static_cast<int64_t>(n_lists) * k > 16384)
    return fail(LD_ERR_INVALID_ARG, "bad merge: %d lists of %d", n_lists, k);
  DevInfo dev;
  int rc = device_info(&dev);
  if (rc) return rc;
  cudaError_t e = launch_merge_peak_lists(peaks, n_peaks, n_lists, k, n_rho, out, n_out,
                                          static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "merge_peak_lists_kernel launch");
  return LD_OK;
}

int ld_bench_smem_atomics(int32_t mode, int32_t iters, int32_t blocks_per_sm,
                          uint64_t *atomics_out, void *scratch, void *stream) {
  g_launches = 0;
  DevInfo dev;
  int rc = device_info(&dev);
  if (rc) return rc;
  if (mode < 0 || mode > 2 || iters < 1 || blocks_per_sm < 1 || !scratch)
    return fail(LD_ERR_INVALID_ARG, "bad microbenchmark arguments");
  const int grid = dev.sm_count * blocks_per_sm;
  cudaError_t e = launch_smem_atomic_bench(mode, iters, grid, static_cast<uint32_t *>(scratch),
                                           static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "smem_atomic_bench_kernel launch");
  if (atomics_out) *atomics_out = static_cast<uint64_t>(grid) * 1024ull * static_cast<uint64_t>(iters);
  return LD_OK;
}

}  // extern "C"
