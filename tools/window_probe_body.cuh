// copied from ld_peaks.cu for tools/window_probe.cu
template <int U, bool NEAR>
__device__ __forceinline__ bool warp_window_max(const uint32_t *A, int64_t ncells, int n_theta,
                                                int n_rho, int t, int r, uint32_t v, int ht,
                                                int hr, int lane) {
  const int idx = t * n_rho + r;
  const int ta = max(t - ht, 0), tb = min(t + ht, n_theta - 1);
  const int ra = max(r - hr, 0), rb = min(r + hr, n_rho - 1);
  const int nc = static_cast<int>(ncells);
  if (NEAR) {
    const int dr = lane - 15;  // lanes 0..30: columns r-15 .. r+15
    const bool col = lane < 31 && r + dr >= ra && r + dr <= rb;
    uint32_t w[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int tt = t - 1 + d;
      w[d] = (col && tt >= ta && tt <= tb) ? __ldg(A + (idx + (d - 1) * n_rho + dr)) : 0u;
    }
    bool bad = false;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      bad |= w[d] > v || (w[d] == v && (d < 1 || (d == 1 && dr < 0))) ||
             (d == 1 && dr == 0 && w[d] != v);
    if (__any_sync(0xffffffffu, bad)) return false;
  }
  {  // the centre row: before r < v, after r <= v, at r == v
    bool bad = false;
    const int row0 = t * n_rho;
#pragma unroll 4
    for (int c = ra + lane; c <= rb; c += 32) {
      const uint32_t w = __ldg(A + row0 + c);
      bad |= c < r ? w >= v : (c > r ? w > v : w != v);  // no short circuit: loads overlap
    }
    if (__any_sync(0xffffffffu, bad)) return false;
  }
  const int rows = tb - ta;  // rows other than the centre one
  if (rows == 0) return true;
  const int nv = (rb - ra + 3) / 4 + 1;  // vectors per row, at any alignment
  const int items = rows * nv;
  const int sh = static_cast<int>((reinterpret_cast<uintptr_t>(A) >> 2) & 3u);  // A's word offset mod 4
  auto row_of = [&](int qq) { return ta + qq + (ta + qq >= t ? 1 : 0); };
  // first cell of the aligned vector holding cell ra of row tt (frame index)
  auto first_vec = [&](int tt) {
    const int c = tt * n_rho + ra;
    return c - ((c + sh) & 3);
  };
  // item 32 u + lane of each step, as (q-th non-centre row, vector j): U
  // independent chains advancing by 32 U items per step
  const int dq = 32 * U / nv, dj = 32 * U - dq * nv;
  int qs[U], js[U], tts[U], a0s[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    qs[u] = (32 * u + lane) / nv;
    js[u] = 32 * u + lane - qs[u] * nv;
    tts[u] = row_of(qs[u]);
    a0s[u] = first_vec(tts[u]);
  }
  uint32_t above = 0u, below = 0u;  // maxima over the rows above / below t
  const int safe = (4 - sh) & 3;  // the frame's first 16-byte-aligned cell
  for (int i0 = 0; i0 < items; i0 += 32 * U) {
    uint4 w[U];
    int lo[U], hi[U], c4[U];  // in-window cells of vector u: e in [lo, hi]
    bool up[U];
    bool edge = false;  // a vector reaching outside the frame's cells
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c4[u] = a0s[u] + 4 * js[u];
      const int col0 = c4[u] - tts[u] * n_rho;
      const bool live = i0 + 32 * u + lane < items && col0 <= rb;
      lo[u] = ra - col0;
      hi[u] = live ? rb - col0 : -1;
      up[u] = tts[u] < t;
      edge |= live && (c4[u] < 0 || c4[u] + 4 > nc);
      if (!live) c4[u] = safe;
      qs[u] += dq;
      js[u] += dj;
      if (js[u] >= nv) {
        js[u] -= nv;
        ++qs[u];
      }
      tts[u] = row_of(qs[u]);
      a0s[u] = first_vec(tts[u]);
    }
    if (!__any_sync(0xffffffffu, edge)) {  // all U vectors of every lane in flight at once
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] = __ldg(reinterpret_cast<const uint4 *>(A + c4[u]));
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c4[u];
        w[u].x = c + 0 >= 0 && c + 0 < nc ? __ldg(A + c + 0) : 0u;
        w[u].y = c + 1 >= 0 && c + 1 < nc ? __ldg(A + c + 1) : 0u;
        w[u].z = c + 2 >= 0 && c + 2 < nc ? __ldg(A + c + 2) : 0u;
        w[u].w = c + 3 >= 0 && c + 3 < nc ? __ldg(A + c + 3) : 0u;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t m01 = max(0 >= lo[u] && 0 <= hi[u] ? w[u].x : 0u,
                               1 >= lo[u] && 1 <= hi[u] ? w[u].y : 0u);
      const uint32_t m23 = max(2 >= lo[u] && 2 <= hi[u] ? w[u].z : 0u,
                               3 >= lo[u] && 3 <= hi[u] ? w[u].w : 0u);
      const uint32_t mv = max(m01, m23);
      above = max(above, up[u] ? mv : 0u);
      below = max(below, up[u] ? 0u : mv);
    }
    if (__any_sync(0xffffffffu, above >= v || below > v)) return false;
  }
  return true;
}
