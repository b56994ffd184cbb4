/*
 * ld.h -- C ABI of libld.so, the B200-native (sm_100a) lane-detection hot path
 * of Alshemi, Saif & Taher, "Hardware Acceleration of Lane Detection
 * Algorithm: a GPU versus FPGA Comparison" (arXiv 2212.09460).
 *
 * The paper's problem statement (Fig. 1): gray 8-bit image -> Sobel
 * edge detection (Step 1) -> binarization (Step 2) -> Hough matrix (Step 3) ->
 * Hough peaks (Step 4, done in MATLAB in the paper).
 * Citations: "P:n" = line n of the paper text; "DESIGN R<k>" = the k-th
 * reading of the paper listed in DESIGN.md section 3.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - All functions are extern "C", never throw, never allocate device memory,
 *    never synchronize the device or the stream.  `stream` is a cudaStream_t
 *    (passed as void*; NULL = legacy default stream).  Work is enqueued on it;
 *    results are valid once the stream reaches that point.  Inputs must stay
 *    unmodified until then.
 *  - Device pointers: every buffer argument is a DEVICE pointer owned by the
 *    caller, except the trig tables (HOST pointers, copied by value into the
 *    launch) and the ld_image descriptor (HOST).  The *_host entry point is
 *    the only one taking host image/peak buffers.
 *  - Outputs are fully overwritten (accumulators zeroed, unused peak slots set
 *    to the sentinel {-1, -1, 0}).
 *  - Validation happens on the host before any launch, so an error status has
 *    no side effect on any output.  On error, ld_last_error_detail() returns a
 *    thread-local one-line explanation.  A failed CUDA call returns
 *    LD_ERR_CUDA and outputs are then undefined.
 *  - Coordinates: origin top-left, x = column, y = row (DESIGN R7).  An edge is
 *    packed as (y << 16) | x in global image coordinates.
 *  - Geometry: D = ceil(sqrt(W^2 + H^2)) (integer), n_rho = 2D + 1 (R10);
 *    theta_t = pi * t / n_theta, t in [0, n_theta) (R8).
 *  - All arithmetic is integer; every output is bit-exact against the oracle.
 */
#ifndef LD_H
#define LD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LD_MAX_DIM 16384   /* W, H <= 16384: x, y fit in 16 bits; rho fits in int32 */
#define LD_MAX_THETA 2048  /* trig tables are passed by value (2 x 8 KB)           */
#define LD_MAX_K 1024      /* peaks per frame                                       */

typedef enum {
  LD_OK = 0,
  LD_ERR_INVALID_ARG = 1, /* null pointer, bad size, misaligned pitch/stride       */
  LD_ERR_RANGE = 2,       /* trig table would put a vote outside [0, n_rho)       */
  LD_ERR_WORKSPACE = 3,   /* workspace too small or misaligned                    */
  LD_ERR_UNSUPPORTED = 4, /* not an sm_100 device, or shared memory too small     */
  LD_ERR_CUDA = 5         /* a CUDA call or launch failed                         */
} ld_status;

/* One Hough peak: signed rho = rho_bin - D.  Sentinel: {-1, -1, 0}. */
typedef struct {
  int32_t theta_bin;
  int32_t rho_bin;
  uint32_t votes;
} ld_peak;

/* A batch of 8-bit gray frames, row-major [batch][rows][pitch] ("a pixel
 * is normally represented by 8 unsigned bits").
 *  width, height : FULL image size; they fix the border, D and coordinates.
 *  pitch         : bytes between rows, >= width, multiple of 16.
 *  frame_stride  : bytes between frames, multiple of 16, >= rows * pitch.
 *  batch         : number of frames, >= 1.
 *  row_begin/end : rows owned by this call, 0 <= row_begin < row_end <= height;
 *                  [0, height) for whole frames, a band for row-banded
 *                  multi-GPU runs.  The gray pointer then addresses global row
 *                  max(row_begin - 1, 0) of frame 0, and rows up to
 *                  min(row_end + 1, height) - 1 must be readable (1-row halo). */
typedef struct {
  int32_t width;
  int32_t height;
  int64_t pitch;
  int64_t frame_stride;
  int32_t batch;
  int32_t row_begin;
  int32_t row_end;
} ld_image;

/* D = ceil(sqrt(W^2 + H^2)) by exact integer square root; -1 if W or H < 1. */
int32_t ld_rho_offset(int32_t width, int32_t height);

/* Steps 1-2 (Eq. 1, Fig. 2; GPU design P:155-169), fused with edge
 * compaction ("threads read the coordinates of input pixels stored in
 * the global memory").  For each owned pixel (x, y):
 *   out = 255 if 1 <= x <= W-2, 1 <= y <= H-2 and |Gx| + |Gy| >= threshold,
 *   out = 0   otherwise (1-px border forced to 0, DESIGN R2; ">=" R4).
 *  threshold   : any int32; <= 0 marks every interior pixel, >= 1531 none.
 *  binary      : nullable. [batch][row_end-row_begin][img->pitch] bytes, output
 *                row i = global row row_begin + i; bytes x >= width are 0.
 *  edge_xy     : nullable. [batch][edge_stride] uint32; frame f's edges are
 *                edge_xy[f*edge_stride + 0 .. edge_count[f]) in UNSPECIFIED
 *                order (a set; DESIGN R15).
 *  edge_stride : >= (row_end-row_begin) * max(width-2, 0) when edge_xy != NULL,
 *                so the list can never overflow.
 *  edge_count  : required. [batch] uint32, overwritten with the edge count.
 * Staging: TMA 2-D tiles with a 1-px halo, persistent CTAs, mbarrier ring. */
int ld_sobel_binarize(const uint8_t *gray, const ld_image *img, int32_t threshold,
                      uint8_t *binary, uint32_t *edge_xy, int64_t edge_stride,
                      uint32_t *edge_count, void *stream);

/* Border / clamp modes of the *_ex entry points (DESIGN
 * R23, R24).  0 = the default of this ABI (1-px output border forced to 0,
 * raw |Gx|+|Gy| compared with T).
 *  LD_FLAG_ZERO_PAD : the paper's own border -- the input is zero-padded by
 *                     one pixel so the output has the input's size (P:106
 *                     FPGA, P:157 GPU): every pixel, border included, is
 *                     filtered with 0 for neighbours outside the image (the
 *                     banded halo rows inside the image stay real rows).
 *  LD_FLAG_CLAMP_255: |G| is clamped to 255 before the threshold (SPEC's 8-bit
 *                     EdgeImage): identical for T <= 255, no edge
 *                     above. */
#define LD_FLAG_ZERO_PAD 1u
#define LD_FLAG_CLAMP_255 2u

/* ld_sobel_binarize with border/clamp flags (any other bit: LD_ERR_INVALID_ARG).
 * With LD_FLAG_ZERO_PAD every owned pixel can be an edge, so edge_stride must
 * be >= (row_end-row_begin) * width. */
int ld_sobel_binarize_ex(const uint8_t *gray, const ld_image *img, int32_t threshold,
                         uint32_t flags, uint8_t *binary, uint32_t *edge_xy,
                         int64_t edge_stride, uint32_t *edge_count, void *stream);

/* Step 3 (Eq. 3; GPU design P:171-175): theta-partitioned voting.
 * acc[f][t][r] = #{ edges e of frame f : ((x*C[t] + y*S[t] + 2^14) >> 15) + D == r }
 * (arithmetic shift = floor; i.e. r - D = round-half-up of x cos + y sin in
 * Q15, DESIGN R9).
 *  edge_xy, edge_count, edge_stride : as produced by ld_sobel_binarize
 *                (DEVICE counts; no host synchronisation is needed).
 *  width, height : full image size (fixes D and n_rho; coordinates must lie
 *                inside it -- true for lists produced by ld_sobel_binarize).
 *  cos_q15, sin_q15 : HOST int32[n_theta], |value| <= 32768, caller supplied
 *                (R11).  Validated: for every t the rho bins of the four image
 *                corners must lie in [0, n_rho), which proves every vote is in
 *                range (rho is linear in x, y and floor is monotone); else
 *                LD_ERR_RANGE.
 *  acc         : [batch][n_theta][n_rho] uint32, fully overwritten.
 * No global atomics: each CTA owns a theta band of the accumulator in shared
 * memory and writes it out with plain coalesced stores. */
int ld_hough_accumulate(const uint32_t *edge_xy, const uint32_t *edge_count,
                        int64_t edge_stride, int32_t batch, int32_t width,
                        int32_t height, int32_t n_theta, const int32_t *cos_q15,
                        const int32_t *sin_q15, uint32_t *acc, void *stream);

/* SPEC's float64 trig mode ("a second, non-bit-exact-vs-Q15
 * workload"; DESIGN R29): ld_hough_accumulate with a HOST
 * double-precision table,
 *   acc[f][t][floor(x*cos[t] + y*sin[t] + 0.5) + D] += 1
 * with each product and each sum rounded to nearest once (no fused
 * multiply-add), so the result is exactly reproducible on any IEEE machine.
 * n_theta <= 1024; entries finite with |value| <= 1; the corner range proof
 * uses the same arithmetic (LD_ERR_RANGE otherwise).  Other arguments as
 * ld_hough_accumulate. */
int ld_hough_accumulate_f64(const uint32_t *edge_xy, const uint32_t *edge_count,
                            int64_t edge_stride, int32_t batch, int32_t width,
                            int32_t height, int32_t n_theta, const double *cos_f64,
                            const double *sin_f64, uint32_t *acc, void *stream);

/* ld_hough_accumulate / ld_hough_accumulate_hint (below) with options:
 *  flags : 0 or any of
 *          LD_VOTE_PLAIN      -- the unpaired voting kernel even for a
 *                                symmetric table (the half-angle pairing of
 *                                Eq. 4-5 is otherwise chosen automatically);
 *          LD_VOTE_NO_CLUSTER -- no thread-block clusters (for launches too
 *                                small to fill the GPU, e.g. one frame, the
 *                                edges of a band are otherwise split over a
 *                                cluster of CTAs whose shared-memory copies
 *                                are summed over distributed shared memory).
 *          Every choice gives the identical accumulator.  Any other bit:
 *          LD_ERR_INVALID_ARG.
 *  hint  : nullable; as ld_hough_accumulate_hint when given. */
#define LD_VOTE_PLAIN 1u
#define LD_VOTE_NO_CLUSTER 2u
int ld_hough_accumulate_opt(const uint32_t *edge_xy, const uint32_t *edge_count,
                            int64_t edge_stride, int32_t batch, int32_t width, int32_t height,
                            int32_t n_theta, const int32_t *cos_q15, const int32_t *sin_q15,
                            uint32_t flags, uint32_t *acc, void *hint, size_t hint_bytes,
                            void *stream);

/* Step 4 ("picking the line with the most pixel value"), made
 * deterministic (DESIGN R13, R14): key(t, r) = (acc[t][r], -t, -r),
 * lexicographic.  (t, r) is a peak candidate iff acc[t][r] >= max(1, min_votes)
 * and its key exceeds every other key in the window |t'-t| <= half_theta,
 * |r'-r| <= half_rho clipped to the accumulator (no theta wrap-around).
 * peaks[f][0..k) = the min(k, #candidates) largest keys, descending, then the
 * sentinel; n_peaks[f] = min(k, #candidates).
 * The search first derives the peak hint of acc into the workspace (one read
 * of acc, as ld_hough_hint_from_acc) and searches only the chunks that can
 * hold a top-k candidate; frames it cannot settle that way go through the
 * dense kernels (LD_PEAKS_DENSE of ld_hough_peaks_opt: those alone).  The
 * result is the same either way.
 *  acc       : [batch][n_theta][n_rho] uint32 (device).
 *  k         : 1..LD_MAX_K.   half_theta, half_rho >= 0.
 *  workspace : device, >= ld_hough_peaks_workspace_bytes(...), 16-B aligned. */
size_t ld_hough_peaks_workspace_bytes(int32_t batch, int32_t n_theta, int32_t n_rho,
                                      int32_t k);
int ld_hough_peaks(const uint32_t *acc, int32_t batch, int32_t n_theta, int32_t n_rho,
                   int32_t half_theta, int32_t half_rho, uint32_t min_votes, int32_t k,
                   ld_peak *peaks, int32_t *n_peaks, void *workspace,
                   size_t workspace_bytes, void *stream);

/* ld_hough_peaks over a theta slice of a larger accumulator (the theta-sharded
 * multi-GPU path): acc holds rows g0 .. g0+n_theta-1 of the
 * full accumulator (theta_offset = g0), including every existing row within
 * half_theta of the candidate rows.  Only cells in rows [cand_row_begin,
 * cand_row_end) (local indices) can be candidates; their windows read any row
 * of acc (clipped to acc, i.e. to the full accumulator when the halo rows are
 * present).  Keys and the reported theta_bin use the global row
 * (local + theta_offset), so per-slice top-k lists merge into the global one
 * exactly.  Requires (theta_offset + n_theta) * n_rho < 2^32 - 1.  An empty
 * row range gives n_peaks = 0. */
int ld_hough_peaks_ex(const uint32_t *acc, int32_t batch, int32_t n_theta, int32_t n_rho,
                      int32_t half_theta, int32_t half_rho, uint32_t min_votes, int32_t k,
                      int32_t cand_row_begin, int32_t cand_row_end, int32_t theta_offset,
                      ld_peak *peaks, int32_t *n_peaks, void *workspace,
                      size_t workspace_bytes, void *stream);

/* Peak hint: an optional by-product of voting that speeds up the peak search
 * without changing its result (DESIGN R25).
 *
 * ld_hough_accumulate_hint votes exactly like ld_hough_accumulate and, while
 * each theta band is still in shared memory, records for each of up to 32
 * contiguous (row-major) ranges of the band the largest count and its cell
 * (value << 32 | ~(t*n_rho + r), i.e. the lowest index among equal counts).
 * ld_hough_peaks_hinted first verifies those cells, largest first, against
 * the candidate definition above (a full window test on acc): verified cells
 * are distinct candidates, so the value of the k-th verified one is a lower
 * bound on the frame's k-th best candidate, and the search starts from it
 * instead of min_votes (a recorded cell also has to hold its recorded value).
 * While each band is in shared memory the voting kernel also records the
 * maximum of every 1 KB chunk (256 counters) of the accumulator's memory;
 * with a certified bound the search then only reads those maxima and tests
 * the cells of the chunks that reach it (the sparse search, DESIGN R30) --
 * bound, sparse search and top k in one kernel per frame -- and falls back to
 * the full search for a frame whose bound is not certified.  peaks / n_peaks
 * are bit-identical to ld_hough_peaks.  The hint must come from the
 * ld_hough_accumulate_hint call that produced acc; a hint whose header
 * (written by that call) does not match batch, n_theta and n_rho is ignored,
 * and the chunk maxima are used only for acc at the address that call wrote
 * (a copy of acc elsewhere gets the full search).
 *  hint : device, >= ld_hough_hint_bytes(batch, width, height, n_theta),
 *         16-B aligned; fully owned by the library between the two calls. */
size_t ld_hough_hint_bytes(int32_t batch, int32_t width, int32_t height, int32_t n_theta);
int ld_hough_accumulate_hint(const uint32_t *edge_xy, const uint32_t *edge_count,
                             int64_t edge_stride, int32_t batch, int32_t width,
                             int32_t height, int32_t n_theta, const int32_t *cos_q15,
                             const int32_t *sin_q15, uint32_t *acc, void *hint,
                             size_t hint_bytes, void *stream);
int ld_hough_peaks_hinted(const uint32_t *acc, int32_t batch, int32_t n_theta, int32_t n_rho,
                          int32_t half_theta, int32_t half_rho, uint32_t min_votes,
                          int32_t k, const void *hint, size_t hint_bytes, ld_peak *peaks,
                          int32_t *n_peaks, void *workspace, size_t workspace_bytes,
                          void *stream);

/* The peak hint of an accumulator that did not come out of one
 * ld_hough_accumulate_hint call -- a sum of partial accumulators after an
 * all_reduce (row-band multi-GPU), a theta shard voted with a slice of the
 * table -- by one read of acc (DESIGN R25, R30): the maximum of every 1 KB
 * chunk of acc's memory and, as range maxima, the best counter of each group
 * of consecutive chunks among candidate rows [cand_row_begin, cand_row_end).
 * Same layout, header and use as the hint of ld_hough_accumulate_hint
 * (ld_hough_peaks_hinted, or ld_hough_peaks_opt with the same candidate rows);
 * it describes acc at this address.  Stream-ordered, no host sync.
 *  acc  : device [batch][n_theta][n_rho] uint32, 4-byte aligned, read only;
 *         n_theta * n_rho < 2^31.
 *  hint : device, >= the ld_hough_hint_bytes of this shape (n_rho =
 *         2 ld_rho_offset(width, height) + 1), 16-B aligned; overwritten.
 * Errors: LD_ERR_INVALID_ARG (NULL pointer, bad shape or rows),
 * LD_ERR_WORKSPACE (hint too small or misaligned). */
int ld_hough_hint_from_acc(const uint32_t *acc, int32_t batch, int32_t n_theta, int32_t n_rho,
                           int32_t cand_row_begin, int32_t cand_row_end, void *hint,
                           size_t hint_bytes, void *stream);

/* The peak search with every option (ld_hough_peaks, _ex and _hinted are
 * this call with defaults): candidate rows and theta offset as
 * ld_hough_peaks_ex; hint nullable (as ld_hough_peaks_hinted; with a
 * restricted row range its keys outside the rows are not used and the sparse
 * search covers those rows only); flags select the search kernels -- every choice
 * returns the same peaks:
 *  LD_PEAKS_DENSE        : no sparse search (DESIGN R30) even with a hint
 *  LD_PEAKS_FORCE_STREAM : the CTA streaming kernel instead of the warp kernel
 *  LD_PEAKS_FORCE_TILE   : the tiled kernel (unrestricted searches only)
 *  LD_PEAKS_FORCE_BAND   : the generic per-cell window scan
 * Any other bit: LD_ERR_INVALID_ARG. */
#define LD_PEAKS_DENSE 1u
#define LD_PEAKS_FORCE_STREAM 2u
#define LD_PEAKS_FORCE_TILE 4u
#define LD_PEAKS_FORCE_BAND 8u
int ld_hough_peaks_opt(const uint32_t *acc, int32_t batch, int32_t n_theta, int32_t n_rho,
                       int32_t half_theta, int32_t half_rho, uint32_t min_votes, int32_t k,
                       int32_t cand_row_begin, int32_t cand_row_end, int32_t theta_offset,
                       const void *hint, size_t hint_bytes, uint32_t flags, ld_peak *peaks,
                       int32_t *n_peaks, void *workspace, size_t workspace_bytes,
                       void *stream);

/* ---------------------------------------------------------------------------
 * Lanes module: Fig. 1 step 4, "draw the
 * lane lines", i.e. MATLAB houghpeaks + houghlines (Fig. 12)
 * made deterministic.  DESIGN R26-R28.
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t x0, y0, x1, y1; /* pixel endpoints, (x0, y0) <= (x1, y1) lexicographically for lines */
} ld_segment;

/* Greedy non-maximum suppression (SPEC find_peaks S:329-337; DESIGN R26):
 * a cell is eligible iff acc >= max(1, min_votes) and
 * acc * ratio_den >= ratio_num * (largest count of the frame); up to k times
 * the eligible, unsuppressed cell with the largest key (acc, -t, -r) is taken
 * and every cell with |t'-t| <= half_theta, |r'-r| <= half_rho (clipped)
 * becomes suppressed.  peaks / n_peaks as ld_hough_peaks (sentinel fill).
 * ratio_den >= 1 (ratio 1/2 = MATLAB's default 0.5 * max).
 *  workspace : device, >= ld_hough_peaks_nms_workspace_bytes(...), 16-B aligned.
 * Cost: k passes over the accumulators (exact for every input). */
size_t ld_hough_peaks_nms_workspace_bytes(int32_t batch, int32_t n_theta, int32_t n_rho);
int ld_hough_peaks_nms(const uint32_t *acc, int32_t batch, int32_t n_theta, int32_t n_rho,
                       int32_t half_theta, int32_t half_rho, uint32_t min_votes,
                       uint32_t ratio_num, uint32_t ratio_den, int32_t k, ld_peak *peaks,
                       int32_t *n_peaks, void *workspace, size_t workspace_bytes,
                       void *stream);

/* peak_to_line (DESIGN R27): for peaks[f][i], i < n_peaks[f],
 * the line x*c + y*s = rho_bin - D with c = C[t]/32768, s = S[t]/32768 (the
 * caller's HOST Q15 table), clipped to the pixel-centre rectangle
 * [0, W-1] x [0, H-1], ends rounded half up; hit[f][i] = 1 and lines[f][i]
 * set, else hit[f][i] = 0 (no intersection, or i >= n_peaks[f]).
 *  peaks [batch][k], n_peaks [batch], lines [batch][k], hit [batch][k]: device. */
int ld_peak_lines(const ld_peak *peaks, const int32_t *n_peaks, int32_t batch, int32_t k,
                  int32_t width, int32_t height, int32_t n_theta, const int32_t *cos_q15,
                  const int32_t *sin_q15, ld_segment *lines, int32_t *hit, void *stream);

/* extract_segments (DESIGN R28): walk the rasterised line of
 * each peak over the binary map (255 = edge): along x when |S[t]| >= |C[t]|,
 * else along y, rounding half up; white samples at most fill_gap + 1 walk
 * steps apart form one run; a run is a segment iff its Euclidean length is
 * >= min_len.  segments[f][i][0..max_segments) in walk order,
 * n_segments[f][i] = how many exist (may exceed max_segments).
 *  binary: device, frames described by img (width, height, pitch,
 *  frame_stride, batch; whole frames), as written by ld_sobel_binarize. */
int ld_extract_segments(const uint8_t *binary, const ld_image *img, const ld_peak *peaks,
                        const int32_t *n_peaks, int32_t k, int32_t n_theta,
                        const int32_t *cos_q15, const int32_t *sin_q15, int32_t fill_gap,
                        int32_t min_len, int32_t max_segments, ld_segment *segments,
                        int32_t *n_segments, void *stream);

/* Steps 1-4 for a batch of whole frames (img->row_begin = 0, row_end = height):
 * ld_sobel_binarize (no binary map) -> ld_hough_accumulate -> ld_hough_peaks,
 * stream-ordered, no host synchronisation.
 *  peaks [batch][k], n_peaks [batch]  : required outputs (device).
 *  edge_count [batch]                 : nullable output (device).
 *  acc [batch][n_theta][n_rho]        : nullable; when given the accumulators
 *                                       are exported there, else they live in
 *                                       the workspace.
 *  workspace : device, >= ld_detect_workspace_bytes(img, n_theta, k, acc==NULL). */
size_t ld_detect_workspace_bytes(const ld_image *img, int32_t n_theta, int32_t k,
                                 int32_t acc_in_workspace);
int ld_detect_batch(const uint8_t *gray, const ld_image *img, int32_t threshold,
                    int32_t n_theta, const int32_t *cos_q15, const int32_t *sin_q15,
                    int32_t half_theta, int32_t half_rho, uint32_t min_votes,
                    int32_t k, ld_peak *peaks, int32_t *n_peaks, uint32_t *edge_count,
                    uint32_t *acc, void *workspace, size_t workspace_bytes,
                    void *stream);

/* ld_detect_batch with border/clamp flags (see LD_FLAG_*); same workspace. */
int ld_detect_batch_ex(const uint8_t *gray, const ld_image *img, int32_t threshold,
                       uint32_t flags, int32_t n_theta, const int32_t *cos_q15,
                       const int32_t *sin_q15, int32_t half_theta, int32_t half_rho,
                       uint32_t min_votes, int32_t k, ld_peak *peaks, int32_t *n_peaks,
                       uint32_t *edge_count, uint32_t *acc, void *workspace,
                       size_t workspace_bytes, void *stream);

/* ld_detect_batch from HOST buffers: gray_host [batch][height][pitch] (pinned
 * host memory for overlap), peaks_host [batch][k], n_peaks_host [batch],
 * edge_count_host [batch] (nullable).  Frames are processed in chunks of
 * chunk_frames: the H2D copy of chunk i+1 overlaps the kernels of chunk i; the
 * D2H copy of peaks/counts is enqueued on `stream`.  Synchronises `stream`
 * before returning (host outputs are valid on return).
 *  workspace : device, >= ld_detect_host_workspace_bytes(img, n_theta, k,
 *              chunk_frames). */
size_t ld_detect_host_workspace_bytes(const ld_image *img, int32_t n_theta, int32_t k,
                                      int32_t chunk_frames);
int ld_detect_batch_host(const uint8_t *gray_host, const ld_image *img,
                         int32_t threshold, int32_t n_theta, const int32_t *cos_q15,
                         const int32_t *sin_q15, int32_t half_theta, int32_t half_rho,
                         uint32_t min_votes, int32_t k, ld_peak *peaks_host,
                         int32_t *n_peaks_host, uint32_t *edge_count_host,
                         int32_t chunk_frames, void *workspace, size_t workspace_bytes,
                         void *stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU helpers of the theta-sharded path (DESIGN
 * section 8; the paper's theta partitioning, lifted across GPUs).  All
 * device-side: no host synchronisation, fixed-size buffers for collectives.
 * ------------------------------------------------------------------------- */
#define LD_MAX_BLOCKS 64 /* row blocks (ranks) of one bitmap */

/* Words of a row-band edge bitmap: rows * ceil(width / 32) uint32. */
int64_t ld_edge_bitmask_words(int32_t width, int32_t rows);

/* The edge set of one row band as a bitmap: bits [rows][ceil(width/32)]
 * (device, 16-B aligned, fully overwritten); bit (x & 31) of word
 * [y - row_begin][x >> 5] is set iff edge (y << 16) | x is in
 * edge_xy[0 .. *edge_count) (device count) and row_begin <= y < row_begin + rows.
 * 1 <= width <= LD_MAX_DIM, rows >= 1. */
int ld_edges_to_bitmask(const uint32_t *edge_xy, const uint32_t *edge_count, int32_t width,
                        int32_t row_begin, int32_t rows, uint32_t *bits, void *stream);

/* The union of n_blocks band bitmaps back to one edge list (order
 * unspecified, a set: DESIGN R15).  bits: device [n_blocks][block_stride_rows]
 * [ceil(width/32)] (the layout an all_gather of equal-size band bitmaps
 * produces); block b holds global rows block_row_begin[b] ..
 * + block_rows[b] - 1 (HOST arrays, block_rows[b] <= block_stride_rows).
 * edge_count (device) receives the number of edges; entries beyond
 * edge_capacity are not written (size the list by the rows: capacity >=
 * sum(block_rows) * width makes overflow impossible).
 * 1 <= n_blocks <= LD_MAX_BLOCKS. */
int ld_bitmask_to_edges(const uint32_t *bits, int32_t width, int32_t n_blocks,
                        const int32_t *block_row_begin, const int32_t *block_rows,
                        int32_t block_stride_rows, uint32_t *edge_xy, int64_t edge_capacity,
                        uint32_t *edge_count, void *stream);

/* The global top k of n_lists top-k lists (peaks [n_lists][k] and n_peaks
 * [n_lists], device; theta_bin global, e.g. the all-gathered results of
 * ld_hough_peaks_ex on theta slices) by the key (votes, -theta, -rho) of
 * DESIGN R14: out [k] (sentinel-filled) and n_out [1], device.  Requires
 * n_lists * k <= 16384 (one CTA sorts them in shared memory). */
int ld_merge_peak_lists(const ld_peak *peaks, const int32_t *n_peaks, int32_t n_lists,
                        int32_t k, int32_t n_rho, ld_peak *out, int32_t *n_out, void *stream);

/* B5 microbenchmark of the shared-memory atomic pipe (the roofline of the
 * voting stage).  Launches one CTA per SM x blocks_per_sm, each thread issuing
 * `iters` red.shared.add.u32 with the given address pattern:
 *   mode 0: conflict-free (lane l always hits bank l, distinct words)
 *   mode 1: pseudo-random addresses over a 48 K-word array
 *   mode 2: one address per warp (fully serialised)
 * *atomics_out (host) receives the total atomics issued.  scratch: device,
 * >= 4 * grid * 34 bytes: per CTA 34 words, 32 checksum words then the clock64
 * cycles of its timed loop (uint64, low word first), so the rate per clock per
 * SM excludes the prologue and the checksum (grid = SMs x blocks_per_sm). */
int ld_bench_smem_atomics(int32_t mode, int32_t iters, int32_t blocks_per_sm,
                          uint64_t *atomics_out, void *scratch, void *stream);

/* Number of SMs / L2 bytes of the current device (host query, cached). */
int32_t ld_device_sm_count(void);
int64_t ld_device_l2_bytes(void);

const char *ld_status_string(int status);
const char *ld_last_error_detail(void);

/* Kernel launches enqueued by the most recent ld_* call on this host thread
 * (for the bench's gpu_launches count). */
int32_t ld_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* LD_H */
