/*
 * ld_oracle.h -- plain, slow, single-threaded CPU oracle of the lane-detection
 * hot path of Alshemi, Saif & Taher, "Hardware Acceleration of Lane Detection
 * Algorithm: a GPU versus FPGA Comparison" (arXiv 2212.09460).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load liboracle.so.  The
 * product path (libld.so and its Python binding) never links, imports or calls
 * anything in oracle/, and this file includes no header of the product.
 *
 * Citations: "P:n" = line n of the paper text (reference PAPER.md);
 * "S:n" = line n of the CPU-program SPEC.md; "DESIGN R<k>" = reading k of the
 * paper listed in DESIGN.md section 3.
 *
 * Every function is pure: it reads its inputs, writes only its outputs, keeps
 * no state, allocates only temporary host memory, and returns 0 on success or a
 * negative LDO_E* code (outputs then undefined).
 *
 * Pins: every function here is pinned by tests/test_oracle_pins.py against
 * hand-computed values, closed forms, library routines and brute force (see
 * DESIGN.md section 4).  No function is "parity unpinned".
 */
#ifndef LD_ORACLE_H
#define LD_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LDO_OK 0
#define LDO_EARG (-1)   /* invalid argument                              */
#define LDO_ERANGE (-2) /* a vote fell outside [0, n_rho) (table too big) */
#define LDO_ECAP (-3)   /* output capacity too small                     */
#define LDO_ENOMEM (-4) /* host malloc failed                            */

typedef struct {
  int32_t theta_bin; /* t in [0, n_theta)                       */
  int32_t rho_bin;   /* r in [0, n_rho); signed rho = r - D     */
  uint32_t votes;    /* acc[t][r]                               */
} ldo_peak;

/* D = ceil(sqrt(W^2 + H^2)), found as the smallest integer D >= 0 with
 * D*D >= W*W + H*H by counting up (no floating point).  n_rho = 2D + 1.
 * DESIGN R10.  Returns -1 for W < 1 or H < 1. */
int32_t ldo_rho_offset(int32_t width, int32_t height);

/* Eq. 1 with the Fig. 2 kernels as correlation weights
 * (row 0 of each kernel multiplies image row y-1; DESIGN R1):
 *   Gx = sum_ij Sx[i][j] * I[y-1+i][x-1+j],  Gy likewise with Sy,
 *   mag[y][x] = |Gx| + |Gy|                      for interior pixels,
 *   mag[y][x] = 0  for x in {0, W-1} or y in {0, H-1} (border, DESIGN R2).
 * gray: [height][pitch] bytes, pitch >= width.  mag: [height][width] int32. */
int ldo_sobel_magnitude(const uint8_t *gray, int32_t width, int32_t height,
                        int64_t pitch, int32_t *mag);

/* Sobel magnitude then binarization:
 *   binary[y][x] = 255 if (interior and |Gx|+|Gy| >= threshold) else 0.
 * The comparison is ">=" on the raw integer magnitude (DESIGN R3, R4).
 * binary: [height][width] bytes. */
int ldo_sobel_binarize(const uint8_t *gray, int32_t width, int32_t height,
                       int64_t pitch, int32_t threshold, uint8_t *binary);

/* Border and clamp modes (DESIGN R23, R24).
 * LDO_ZERO_PAD: the paper's own border -- "zero padding" of the input so the
 *   output has the input's size (P:106 FPGA, P:157 GPU): every
 *   pixel, border included, is filtered, with 0 for neighbours outside.
 * LDO_CLAMP_255: |G| is clamped to 255 before the threshold, SPEC's 8-bit
 *   EdgeImage.
 * ldo_sobel_magnitude_ex writes the (unclamped) magnitude under the border
 * mode of `flags`; ldo_sobel_binarize_ex binarizes it with ">=" (R4), applying
 * the clamp when asked.  flags = 0 is exactly ldo_sobel_binarize. */
#define LDO_ZERO_PAD 1
#define LDO_CLAMP_255 2
int ldo_sobel_magnitude_ex(const uint8_t *gray, int32_t width, int32_t height,
                           int64_t pitch, int32_t flags, int32_t *mag);
int ldo_sobel_binarize_ex(const uint8_t *gray, int32_t width, int32_t height,
                          int64_t pitch, int32_t threshold, int32_t flags,
                          uint8_t *binary);

/* Edge-coordinate list ("threads read the coordinates of input pixels
 * stored in the global memory"): raster scan (y-major, then x) of binary
 * [height][width]; appends (y << 16) | x for every pixel equal to 255.
 * Writes *n_edges.  Returns LDO_ECAP if more than cap edges. */
int ldo_compact(const uint8_t *binary, int32_t width, int32_t height,
                uint32_t *edges, int64_t cap, int64_t *n_edges);

/* Hough voting (Eq. 3; DESIGN R8, R9, R11, R12).
 * acc[n_theta][n_rho] (n_rho = 2D+1) is zeroed, then for every edge (x, y)
 * and every t in [0, n_theta):
 *   v   = x*C[t] + y*S[t] + 2^14           (64-bit integer)
 *   rho = floor(v / 2^15) + D              (explicit floor division)
 *   acc[t][rho] += 1
 * i.e. rho - D is r = x cos(theta_t) + y sin(theta_t) in Q15 rounded half up.
 * Returns LDO_ERANGE (acc undefined) if any rho leaves [0, n_rho). */
int ldo_hough_accumulate(const uint32_t *edges, int64_t n_edges, int32_t width,
                         int32_t height, int32_t n_theta, const int32_t *cos_q15,
                         const int32_t *sin_q15, uint32_t *acc);

/* SPEC's float64 trig mode ("a second, non-bit-exact-
 * vs-Q15 workload"; DESIGN R29): the same voting with the caller's
 * double-precision table,
 *   r   = x*cos[t] + y*sin[t]   (each product and the sum rounded once)
 *   rho = floor(r + 0.5) + D    (S:224 quantize = round half up)
 *   acc[t][rho] += 1.
 * Returns LDO_ERANGE (acc undefined) if any rho leaves [0, n_rho). */
int ldo_hough_accumulate_f64(const uint32_t *edges, int64_t n_edges, int32_t width,
                             int32_t height, int32_t n_theta, const double *cos_f64,
                             const double *sin_f64, uint32_t *acc);

/* Hough peaks ("picking the line with the most pixel value"; P:185;
 * DESIGN R13, R14).  key(t, r) = (acc[t][r], -t, -r), compared
 * lexicographically.  (t, r) is a candidate iff
 *   acc[t][r] >= max(1, min_votes)  and
 *   key(t, r) > key(t', r') for every other (t', r') with |t'-t| <= half_theta,
 *   |r'-r| <= half_rho, inside the accumulator (no theta wrap-around).
 * Candidates are sorted by key, descending; the first min(k, #candidates) are
 * written to peaks[0..), the rest of peaks[0..k) is {-1, -1, 0}.
 * *n_peaks = min(k, #candidates). */
int ldo_hough_peaks(const uint32_t *acc, int32_t n_theta, int32_t n_rho,
                    int32_t half_theta, int32_t half_rho, uint32_t min_votes,
                    int32_t k, ldo_peak *peaks, int32_t *n_peaks);

/* The whole per-frame pipeline (Fig. 1 steps 1-3 plus the peak step):
 * sobel_binarize -> compact -> hough_accumulate -> hough_peaks.
 * binary (nullable) [height][width]; acc (nullable) [n_theta][2D+1];
 * edges (nullable) [width*height], raster order; n_edges required. */
int ldo_detect(const uint8_t *gray, int32_t width, int32_t height, int64_t pitch,
               int32_t threshold, int32_t n_theta, const int32_t *cos_q15,
               const int32_t *sin_q15, int32_t half_theta, int32_t half_rho,
               uint32_t min_votes, int32_t k, uint8_t *binary, uint32_t *edges,
               int64_t *n_edges, uint32_t *acc, ldo_peak *peaks,
               int32_t *n_peaks);

/* ---------------------------------------------------------------------------
 * NEXT 3: SPEC's lanes module, completing Fig. 1 step 4 (P:42,
 * "draw the lane lines"; P:185 MATLAB houghpeaks / Fig. 12 houghlines).
 * DESIGN R26-R28.
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t x0, y0, x1, y1; /* pixel endpoints */
} ldo_segment;

/* R26, SPEC find_peaks: greedy non-maximum suppression.
 *   gmax = the largest count of acc; a cell is eligible iff
 *     acc >= max(1, min_votes)  and  acc * ratio_den >= ratio_num * gmax
 *   (the "threshold_ratio x global max" rule as an exact integer test);
 *   repeat up to k times: select the eligible, not yet suppressed cell with
 *   the largest key(t, r) = (acc, -t, -r); stop if there is none; suppress
 *   every cell with |t'-t| <= half_theta and |r'-r| <= half_rho (clipped, no
 *   theta wrap-around), the selected cell included.
 * peaks[0..k) and *n_peaks as ldo_hough_peaks (sentinel {-1,-1,0} fill).
 * ratio_den >= 1. */
int ldo_hough_peaks_nms(const uint32_t *acc, int32_t n_theta, int32_t n_rho,
                        int32_t half_theta, int32_t half_rho, uint32_t min_votes,
                        uint32_t ratio_num, uint32_t ratio_den, int32_t k,
                        ldo_peak *peaks, int32_t *n_peaks);

/* R27, SPEC peak_to_line: the line x*c + y*s = rho of a peak,
 * c = C[t] / 32768, s = S[t] / 32768 (the caller's Q15 table, exact binary
 * fractions), rho = rho_bin - D, clipped to the rectangle of pixel centres
 * [0, W-1] x [0, H-1].  In double precision, each product and quotient
 * rounded once (no fused multiply-add):
 *   for X in {0, W-1}, if s != 0: Y = (rho - X*c) / s, kept if 0 <= Y <= H-1;
 *   for Y in {0, H-1}, if c != 0: X = (rho - Y*s) / c, kept if 0 <= X <= W-1;
 *   the kept points with the smallest and the largest projection -X*s + Y*c
 *   (first one found on ties) are the ends; each coordinate is rounded to
 *   floor(v + 0.5); seg = the two ends, the lexicographically smaller (x, y)
 *   first.  *hit = 0 (seg untouched) when no point is kept. */
int ldo_peak_to_line(ldo_peak peak, int32_t width, int32_t height, int32_t n_theta,
                     const int32_t *cos_q15, const int32_t *sin_q15, ldo_segment *seg,
                     int32_t *hit);

/* R28, SPEC extract_segments: walk the rasterised peak line
 * (c, s, rho as in R27).  If |S[t]| >= |C[t]| the walk steps x = 0 .. W-1
 * with y = floor((rho - x*c) / s + 0.5), else y = 0 .. H-1 with
 * x = floor((rho - y*s) / c + 0.5); a sample is white iff it lies in the
 * image and binary == 255.  White samples whose walk indices differ by at
 * most fill_gap + 1 belong to one run; a run from sample a to sample b is a
 * segment (a, b) iff (xb-xa)^2 + (yb-ya)^2 >= min_len^2.  Segments in walk
 * order; the first cap are written, *n_segs = how many there are.  A table
 * entry with C[t] = S[t] = 0 has no line: *n_segs = 0. */
int ldo_extract_segments(const uint8_t *binary, int32_t width, int32_t height,
                         int64_t pitch, ldo_peak peak, int32_t n_theta,
                         const int32_t *cos_q15, const int32_t *sin_q15,
                         int32_t fill_gap, int32_t min_len, ldo_segment *segs,
                         int32_t cap, int32_t *n_segs);

#ifdef __cplusplus
}
#endif
#endif /* LD_ORACLE_H */
