/*
 * ld_oracle.c -- plain single-threaded C99 oracle for the lane-detection hot
 * path of arXiv 2212.09460.  TEST INFRASTRUCTURE ONLY (see ld_oracle.h): it is
 * written for a reader checking it against the paper by eye, not for speed.
 * No blocking, fusion, vectorisation or reordering beyond the paper's own
 * definitions; it shares no code, header or table with the CUDA path.
 */
#include "ld_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Fig. 2: the two Sobel kernels, row 0 on top. */
static const int SOBEL_X[3][3] = {{-1, 0, +1}, {-2, 0, +2}, {-1, 0, +1}};
static const int SOBEL_Y[3][3] = {{+1, +2, +1}, {0, 0, 0}, {-1, -2, -1}};

int32_t ldo_rho_offset(int32_t width, int32_t height) {
  if (width < 1 || height < 1) return -1;
  int64_t d2 = (int64_t)width * width + (int64_t)height * height;
  int64_t d = 0;
  while (d * d < d2) d++; /* smallest D with D^2 >= W^2 + H^2 */
  return (int32_t)d;
}

static int32_t iabs32(int32_t v) { return v < 0 ? -v : v; }

int ldo_sobel_magnitude(const uint8_t *gray, int32_t width, int32_t height,
                        int64_t pitch, int32_t *mag) {
  if (!gray || !mag || width < 1 || height < 1 || pitch < width) return LDO_EARG;
  for (int32_t y = 0; y < height; y++) {
    for (int32_t x = 0; x < width; x++) {
      int border = (x == 0 || x == width - 1 || y == 0 || y == height - 1);
      if (border) { /* DESIGN R2: 1-px output border forced to 0 */
        mag[(int64_t)y * width + x] = 0;
        continue;
      }
      int32_t gx = 0, gy = 0; /* Eq. 1: literal multiply-accumulate */
      for (int i = 0; i < 3; i++) {
        for (int j = 0; j < 3; j++) {
          int32_t p = gray[(int64_t)(y - 1 + i) * pitch + (x - 1 + j)];
          gx += SOBEL_X[i][j] * p;
          gy += SOBEL_Y[i][j] * p;
        }
      }
      mag[(int64_t)y * width + x] = iabs32(gx) + iabs32(gy);
    }
  }
  return LDO_OK;
}

int ldo_sobel_binarize(const uint8_t *gray, int32_t width, int32_t height,
                       int64_t pitch, int32_t threshold, uint8_t *binary) {
  if (!gray || !binary || width < 1 || height < 1 || pitch < width) return LDO_EARG;
  int32_t *mag = (int32_t *)malloc(sizeof(int32_t) * (size_t)width * (size_t)height);
  if (!mag) return LDO_ENOMEM;
  int rc = ldo_sobel_magnitude(gray, width, height, pitch, mag);
  if (rc == LDO_OK) {
    for (int32_t y = 0; y < height; y++) {
      for (int32_t x = 0; x < width; x++) {
        int64_t i = (int64_t)y * width + x;
        int border = (x == 0 || x == width - 1 || y == 0 || y == height - 1);
        /* P:76 every pixel becomes 255 or 0; comparator sense ">=" (R4) */
        binary[i] = (!border && mag[i] >= threshold) ? 255 : 0;
      }
    }
  }
  free(mag);
  return rc;
}

int ldo_sobel_magnitude_ex(const uint8_t *gray, int32_t width, int32_t height,
                           int64_t pitch, int32_t flags, int32_t *mag) {
  if (!(flags & LDO_ZERO_PAD)) return ldo_sobel_magnitude(gray, width, height, pitch, mag);
  if (!gray || !mag || width < 1 || height < 1 || pitch < width) return LDO_EARG;
  for (int32_t y = 0; y < height; y++) {
    for (int32_t x = 0; x < width; x++) {
      int32_t gx = 0, gy = 0; /* Eq. 1 on the zero-padded image */
      for (int i = 0; i < 3; i++) {
        for (int j = 0; j < 3; j++) {
          int32_t yy = y - 1 + i, xx = x - 1 + j;
          int32_t p = (yy < 0 || yy >= height || xx < 0 || xx >= width)
                          ? 0
                          : gray[(int64_t)yy * pitch + xx];
          gx += SOBEL_X[i][j] * p;
          gy += SOBEL_Y[i][j] * p;
        }
      }
      mag[(int64_t)y * width + x] = iabs32(gx) + iabs32(gy);
    }
  }
  return LDO_OK;
}

int ldo_sobel_binarize_ex(const uint8_t *gray, int32_t width, int32_t height,
                          int64_t pitch, int32_t threshold, int32_t flags,
                          uint8_t *binary) {
  if (!(flags & LDO_ZERO_PAD) && !(flags & LDO_CLAMP_255))
    return ldo_sobel_binarize(gray, width, height, pitch, threshold, binary);
  if (!gray || !binary || width < 1 || height < 1 || pitch < width) return LDO_EARG;
  int32_t *mag = (int32_t *)malloc(sizeof(int32_t) * (size_t)width * (size_t)height);
  if (!mag) return LDO_ENOMEM;
  int rc = ldo_sobel_magnitude_ex(gray, width, height, pitch, flags, mag);
  if (rc == LDO_OK) {
    for (int32_t y = 0; y < height; y++) {
      for (int32_t x = 0; x < width; x++) {
        int64_t i = (int64_t)y * width + x;
        int32_t g = mag[i];
        if ((flags & LDO_CLAMP_255) && g > 255) g = 255;
        int border = (x == 0 || x == width - 1 || y == 0 || y == height - 1);
        int forced0 = border && !(flags & LDO_ZERO_PAD); /* R2 unless zero-padded */
        binary[i] = (!forced0 && g >= threshold) ? 255 : 0;
      }
    }
  }
  free(mag);
  return rc;
}

int ldo_compact(const uint8_t *binary, int32_t width, int32_t height,
                uint32_t *edges, int64_t cap, int64_t *n_edges) {
  if (!binary || !n_edges || width < 1 || height < 1 || width > 65536 ||
      height > 65536 || cap < 0 || (cap > 0 && !edges))
    return LDO_EARG;
  int64_t n = 0;
  for (int32_t y = 0; y < height; y++) {
    for (int32_t x = 0; x < width; x++) {
      if (binary[(int64_t)y * width + x] == 255) {
        if (n >= cap) return LDO_ECAP;
        edges[n++] = ((uint32_t)y << 16) | (uint32_t)x;
      }
    }
  }
  *n_edges = n;
  return LDO_OK;
}

/* floor(a / b) for b > 0, written with C division (which truncates toward 0)
 * and an explicit correction -- deliberately not an arithmetic shift. */
static int64_t floor_div(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
  return q;
}

int ldo_hough_accumulate(const uint32_t *edges, int64_t n_edges, int32_t width,
                         int32_t height, int32_t n_theta, const int32_t *cos_q15,
                         const int32_t *sin_q15, uint32_t *acc) {
  if (!acc || !cos_q15 || !sin_q15 || n_theta < 1 || n_edges < 0 ||
      (n_edges > 0 && !edges))
    return LDO_EARG;
  int32_t d = ldo_rho_offset(width, height);
  if (d < 0) return LDO_EARG;
  int64_t n_rho = 2 * (int64_t)d + 1;
  memset(acc, 0, sizeof(uint32_t) * (size_t)n_theta * (size_t)n_rho);
  for (int64_t e = 0; e < n_edges; e++) {
    int64_t x = edges[e] & 0xFFFFu;
    int64_t y = edges[e] >> 16;
    if (x >= width || y >= height) return LDO_EARG;
    for (int32_t t = 0; t < n_theta; t++) {
      /* Eq. 3: r = x cos(theta) + y sin(theta), Q15, rounded half up */
      int64_t v = x * cos_q15[t] + y * sin_q15[t] + 16384;
      int64_t rho = floor_div(v, 32768) + d;
      if (rho < 0 || rho >= n_rho) return LDO_ERANGE;
      acc[(int64_t)t * n_rho + rho] += 1;
    }
  }
  return LDO_OK;
}

/* key(a) > key(b) with key = (votes, -theta, -rho) */
static int key_greater(uint32_t va, int32_t ta, int32_t ra, uint32_t vb,
                       int32_t tb, int32_t rb) {
  if (va != vb) return va > vb;
  if (ta != tb) return ta < tb;
  return ra < rb;
}

static int peak_cmp_desc(const void *pa, const void *pb) {
  const ldo_peak *a = (const ldo_peak *)pa, *b = (const ldo_peak *)pb;
  if (key_greater(a->votes, a->theta_bin, a->rho_bin, b->votes, b->theta_bin,
                  b->rho_bin))
    return -1;
  if (key_greater(b->votes, b->theta_bin, b->rho_bin, a->votes, a->theta_bin,
                  a->rho_bin))
    return 1;
  return 0;
}

int ldo_hough_peaks(const uint32_t *acc, int32_t n_theta, int32_t n_rho,
                    int32_t half_theta, int32_t half_rho, uint32_t min_votes,
                    int32_t k, ldo_peak *peaks, int32_t *n_peaks) {
  if (!acc || !peaks || !n_peaks || n_theta < 1 || n_rho < 1 ||
      half_theta < 0 || half_rho < 0 || k < 1)
    return LDO_EARG;
  uint32_t floor_votes = min_votes > 1 ? min_votes : 1;
  int64_t cap = 1024, count = 0;
  ldo_peak *cand = (ldo_peak *)malloc(sizeof(ldo_peak) * (size_t)cap);
  if (!cand) return LDO_ENOMEM;
  for (int32_t t = 0; t < n_theta; t++) {
    for (int32_t r = 0; r < n_rho; r++) {
      uint32_t v = acc[(int64_t)t * n_rho + r];
      if (v < floor_votes) continue;
      int is_max = 1;
      /* window N(t, r), clipped to the accumulator, no theta wrap-around */
      for (int32_t tt = t - half_theta; tt <= t + half_theta && is_max; tt++) {
        if (tt < 0 || tt >= n_theta) continue;
        for (int32_t rr = r - half_rho; rr <= r + half_rho; rr++) {
          if (rr < 0 || rr >= n_rho || (tt == t && rr == r)) continue;
          uint32_t w = acc[(int64_t)tt * n_rho + rr];
          if (!key_greater(v, t, r, w, tt, rr)) { is_max = 0; break; }
        }
      }
      if (!is_max) continue;
      if (count == cap) {
        cap *= 2;
        ldo_peak *grown = (ldo_peak *)realloc(cand, sizeof(ldo_peak) * (size_t)cap);
        if (!grown) { free(cand); return LDO_ENOMEM; }
        cand = grown;
      }
      cand[count].theta_bin = t;
      cand[count].rho_bin = r;
      cand[count].votes = v;
      count++;
    }
  }
  qsort(cand, (size_t)count, sizeof(ldo_peak), peak_cmp_desc);
  int32_t m = count < k ? (int32_t)count : k;
  for (int32_t i = 0; i < k; i++) {
    if (i < m) {
      peaks[i] = cand[i];
    } else {
      peaks[i].theta_bin = -1;
      peaks[i].rho_bin = -1;
      peaks[i].votes = 0;
    }
  }
  *n_peaks = m;
  free(cand);
  return LDO_OK;
}

int ldo_detect(const uint8_t *gray, int32_t width, int32_t height, int64_t pitch,
               int32_t threshold, int32_t n_theta, const int32_t *cos_q15,
               const int32_t *sin_q15, int32_t half_theta, int32_t half_rho,
               uint32_t min_votes, int32_t k, uint8_t *binary, uint32_t *edges,
               int64_t *n_edges, uint32_t *acc, ldo_peak *peaks,
               int32_t *n_peaks) {
  if (!gray || !n_edges || !peaks || !n_peaks || width < 1 || height < 1 ||
      n_theta < 1)
    return LDO_EARG;
  int32_t d = ldo_rho_offset(width, height);
  int64_t n_rho = 2 * (int64_t)d + 1;
  size_t npx = (size_t)width * (size_t)height;
  uint8_t *bin = binary ? binary : (uint8_t *)malloc(npx);
  uint32_t *edg = edges ? edges : (uint32_t *)malloc(sizeof(uint32_t) * npx);
  uint32_t *ac = acc ? acc : (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n_theta * (size_t)n_rho);
  int rc = LDO_ENOMEM;
  if (bin && edg && ac) {
    rc = ldo_sobel_binarize(gray, width, height, pitch, threshold, bin);
    if (rc == LDO_OK) rc = ldo_compact(bin, width, height, edg, (int64_t)npx, n_edges);
    if (rc == LDO_OK)
      rc = ldo_hough_accumulate(edg, *n_edges, width, height, n_theta, cos_q15,
                                sin_q15, ac);
    if (rc == LDO_OK)
      rc = ldo_hough_peaks(ac, n_theta, (int32_t)n_rho, half_theta, half_rho,
                           min_votes, k, peaks, n_peaks);
  }
  if (!binary) free(bin);
  if (!edges) free(edg);
  if (!acc) free(ac);
  return rc;
}

/* ---------------------------------------------------------------------------
 * NEXT 3: lanes module (R26-R28)
 * ------------------------------------------------------------------------- */
int ldo_hough_peaks_nms(const uint32_t *acc, int32_t n_theta, int32_t n_rho,
                        int32_t half_theta, int32_t half_rho, uint32_t min_votes,
                        uint32_t ratio_num, uint32_t ratio_den, int32_t k,
                        ldo_peak *peaks, int32_t *n_peaks) {
  if (!acc || !peaks || !n_peaks || n_theta < 1 || n_rho < 1 || half_theta < 0 ||
      half_rho < 0 || k < 1 || ratio_den < 1)
    return LDO_EARG;
  const int64_t cells = (int64_t)n_theta * n_rho;
  uint32_t gmax = 0;
  for (int64_t i = 0; i < cells; i++)
    if (acc[i] > gmax) gmax = acc[i];
  uint32_t floor_votes = min_votes > 1 ? min_votes : 1;
  unsigned char *suppressed = (unsigned char *)calloc((size_t)cells, 1);
  if (!suppressed) return LDO_ENOMEM;
  int32_t m = 0;
  while (m < k) {
    /* the eligible, unsuppressed cell with the largest key */
    int64_t best = -1;
    for (int32_t t = 0; t < n_theta; t++) {
      for (int32_t r = 0; r < n_rho; r++) {
        int64_t i = (int64_t)t * n_rho + r;
        uint32_t v = acc[i];
        if (suppressed[i] || v < floor_votes) continue;
        if ((uint64_t)v * ratio_den < (uint64_t)ratio_num * gmax) continue;
        if (best < 0 || key_greater(v, t, r, acc[best], (int32_t)(best / n_rho),
                                    (int32_t)(best % n_rho)))
          best = i;
      }
    }
    if (best < 0) break;
    int32_t bt = (int32_t)(best / n_rho), br = (int32_t)(best % n_rho);
    peaks[m].theta_bin = bt;
    peaks[m].rho_bin = br;
    peaks[m].votes = acc[best];
    m++;
    for (int32_t t = bt - half_theta; t <= bt + half_theta; t++) {
      if (t < 0 || t >= n_theta) continue;
      for (int32_t r = br - half_rho; r <= br + half_rho; r++) {
        if (r < 0 || r >= n_rho) continue;
        suppressed[(int64_t)t * n_rho + r] = 1;
      }
    }
  }
  for (int32_t i = m; i < k; i++) {
    peaks[i].theta_bin = -1;
    peaks[i].rho_bin = -1;
    peaks[i].votes = 0;
  }
  *n_peaks = m;
  free(suppressed);
  return LDO_OK;
}

static int32_t round_half_up(double v) { return (int32_t)floor(v + 0.5); }

int ldo_peak_to_line(ldo_peak peak, int32_t width, int32_t height, int32_t n_theta,
                     const int32_t *cos_q15, const int32_t *sin_q15, ldo_segment *seg,
                     int32_t *hit) {
  if (!cos_q15 || !sin_q15 || !seg || !hit || width < 1 || height < 1 ||
      peak.theta_bin < 0 || peak.theta_bin >= n_theta)
    return LDO_EARG;
  int32_t d = ldo_rho_offset(width, height);
  double c = (double)cos_q15[peak.theta_bin] / 32768.0;
  double s = (double)sin_q15[peak.theta_bin] / 32768.0;
  double rho = (double)(peak.rho_bin - d);
  double px[4], py[4];
  int n = 0;
  double xs[2] = {0.0, (double)(width - 1)}, ys[2] = {0.0, (double)(height - 1)};
  if (s != 0.0) {
    for (int i = 0; i < 2; i++) {
      double y = (rho - xs[i] * c) / s;
      if (y >= 0.0 && y <= (double)(height - 1)) { px[n] = xs[i]; py[n] = y; n++; }
    }
  }
  if (c != 0.0) {
    for (int i = 0; i < 2; i++) {
      double x = (rho - ys[i] * s) / c;
      if (x >= 0.0 && x <= (double)(width - 1)) { px[n] = x; py[n] = ys[i]; n++; }
    }
  }
  if (n == 0) { *hit = 0; return LDO_OK; }
  int lo = 0, hi = 0;
  double plo = -px[0] * s + py[0] * c, phi = plo;
  for (int i = 1; i < n; i++) {
    double p = -px[i] * s + py[i] * c;
    if (p < plo) { plo = p; lo = i; }
    if (p > phi) { phi = p; hi = i; }
  }
  int32_t ax = round_half_up(px[lo]), ay = round_half_up(py[lo]);
  int32_t bx = round_half_up(px[hi]), by = round_half_up(py[hi]);
  if (bx < ax || (bx == ax && by < ay)) {
    int32_t tx = ax, ty = ay;
    ax = bx; ay = by; bx = tx; by = ty;
  }
  seg->x0 = ax; seg->y0 = ay; seg->x1 = bx; seg->y1 = by;
  *hit = 1;
  return LDO_OK;
}

int ldo_extract_segments(const uint8_t *binary, int32_t width, int32_t height,
                         int64_t pitch, ldo_peak peak, int32_t n_theta,
                         const int32_t *cos_q15, const int32_t *sin_q15,
                         int32_t fill_gap, int32_t min_len, ldo_segment *segs,
                         int32_t cap, int32_t *n_segs) {
  if (!binary || !cos_q15 || !sin_q15 || !n_segs || width < 1 || height < 1 ||
      pitch < width || peak.theta_bin < 0 || peak.theta_bin >= n_theta ||
      fill_gap < 0 || min_len < 0 || cap < 0 || (cap > 0 && !segs))
    return LDO_EARG;
  int32_t d = ldo_rho_offset(width, height);
  int32_t ci = cos_q15[peak.theta_bin], si = sin_q15[peak.theta_bin];
  *n_segs = 0;
  if (ci == 0 && si == 0) return LDO_OK;
  double c = (double)ci / 32768.0, s = (double)si / 32768.0;
  double rho = (double)(peak.rho_bin - d);
  int along_x = (si < 0 ? -si : si) >= (ci < 0 ? -ci : ci);
  int32_t n = along_x ? width : height;
  int32_t count = 0;
  int32_t run_a = -1, run_b = -1; /* walk indices of the current run's ends */
  int32_t ax = 0, ay = 0, bx = 0, by = 0;
  for (int32_t i = 0; i <= n; i++) {
    int white = 0;
    int32_t x = 0, y = 0;
    if (i < n) {
      if (along_x) { x = i; y = round_half_up((rho - (double)i * c) / s); }
      else { y = i; x = round_half_up((rho - (double)i * s) / c); }
      white = x >= 0 && x < width && y >= 0 && y < height &&
              binary[(int64_t)y * pitch + x] == 255;
    }
    /* close the run when the walk ends or this white sample is too far */
    if (run_a >= 0 && (i == n || (white && i - run_b - 1 > fill_gap))) {
      int64_t dx = bx - ax, dy = by - ay;
      if (dx * dx + dy * dy >= (int64_t)min_len * min_len) {
        if (count < cap) {
          segs[count].x0 = ax; segs[count].y0 = ay;
          segs[count].x1 = bx; segs[count].y1 = by;
        }
        count++;
      }
      run_a = -1;
    }
    if (!white) continue;
    if (run_a < 0) { run_a = i; ax = x; ay = y; }
    run_b = i; bx = x; by = y;
  }
  *n_segs = count;
  return LDO_OK;
}

int ldo_hough_accumulate_f64(const uint32_t *edges, int64_t n_edges, int32_t width,
                             int32_t height, int32_t n_theta, const double *cos_f64,
                             const double *sin_f64, uint32_t *acc) {
  if ((!edges && n_edges > 0) || !cos_f64 || !sin_f64 || !acc || n_edges < 0 || width < 1 ||
      height < 1 || n_theta < 1)
    return LDO_EARG;
  int32_t d = ldo_rho_offset(width, height);
  int64_t n_rho = 2 * (int64_t)d + 1;
  memset(acc, 0, sizeof(uint32_t) * (size_t)n_theta * (size_t)n_rho);
  for (int64_t i = 0; i < n_edges; i++) {
    double x = (double)(edges[i] & 0xFFFFu), y = (double)(edges[i] >> 16);
    for (int32_t t = 0; t < n_theta; t++) {
      double px = x * cos_f64[t];
      double py = y * sin_f64[t];
      double r = px + py;
      int64_t rho = (int64_t)floor(r + 0.5) + d;
      if (rho < 0 || rho >= n_rho) return LDO_ERANGE;
      acc[(int64_t)t * n_rho + rho] += 1;
    }
  }
  return LDO_OK;
}
