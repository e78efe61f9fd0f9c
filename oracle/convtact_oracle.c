/*
 * convtact_oracle.c -- CPU restatement of the reference convtact hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and there only as
 * the checker or the timed CPU baseline -- never as the product path.
 *
 * Each function restates the float64 algorithm of the reference package
 * /root/reference/pkg/src/convtact (cited file:line), keeping its per-element
 * summation order so results agree with the reference to the last ulp:
 *   - direct correlation: taps accumulated in row-major order from 0.0 with
 *     fused multiply-add (numba @njit(fastmath=True) contracts
 *     `out += kv * s` into FMA on FMA hardware, _loops.py:27-198);
 *   - numpy elementwise expressions are evaluated op by op without
 *     contraction (this file is compiled with -ffp-contract=off);
 *   - np.sum over a contiguous temporary is numpy's pairwise summation
 *     (8-way unrolled blocks of <=128, recursive halving), restated exactly
 *     in pairwise_sum() below.
 * Parity is pinned by tests/test_oracle_golden.py against fixtures generated
 * by running the reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MAXDIM 32

/* ---------------------------------------------------------------- conv --- */

/* Zero-extended correlation for any rank: out[o] = sum_j k[j] * s[o - pl + j]
 * over in-range taps only, taps in row-major order.  This is the per-element
 * semantics of _loops.xcorr_zpad_{1,2,3}d (_loops.py:72-198) and of the
 * pad-then-shift-and-add path for ndim >= 4 (conv.py:128-130,
 * _loops.py:201-208).  The loop nest keeps the reference's row-blocked order
 * (output row, then taps, innermost contiguous x).  Ranks 1-3 run numba loops
 * that contract to FMA; ranks >= 4 run numpy `out += k[idx] * s[window]`,
 * a rounded product then a rounded add. */
static void xcorr_rows(int ndim, const double* s, const int64_t* ms, const int64_t* sstr,
                       const double* k, const int64_t* ns, const int64_t* kstr,
                       const int64_t* pl, const int64_t* os, double* out) {
  const int last = ndim - 1;
  const int fused = ndim <= 3;
  int64_t nrows = 1, ntaps_outer = 1;
  for (int d = 0; d < last; ++d) { nrows *= os[d]; ntaps_outer *= ns[d]; }
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t oidx[OR_MAXDIM];
    int64_t rem = r;
    for (int d = last - 1; d >= 0; --d) { oidx[d] = rem % os[d]; rem /= os[d]; }
    double* orow = out + r * os[last];
    for (int64_t t = 0; t < ntaps_outer; ++t) {
      int64_t jidx[OR_MAXDIM];
      int64_t trem = t;
      for (int d = last - 1; d >= 0; --d) { jidx[d] = trem % ns[d]; trem /= ns[d]; }
      int64_t soff = 0, koff = 0;
      int inb = 1;
      for (int d = 0; d < last; ++d) {
        const int64_t si = oidx[d] - pl[d] + jidx[d];
        if (si < 0 || si >= ms[d]) { inb = 0; break; }
        soff += si * sstr[d];
        koff += jidx[d] * kstr[d];
      }
      if (!inb) continue;
      for (int64_t j = 0; j < ns[last]; ++j) {
        const double kv = k[koff + j];
        const int64_t dd = j - pl[last];
        const int64_t lo = -dd > 0 ? -dd : 0;
        const int64_t hi = ms[last] - dd < os[last] ? ms[last] - dd : os[last];
        const double* srow = s + soff + dd;
        if (fused) {
          for (int64_t x = lo; x < hi; ++x) orow[x] = fma(kv, srow[x], orow[x]);
        } else {
          for (int64_t x = lo; x < hi; ++x) {
            const double p = kv * srow[x];
            orow[x] = orow[x] + p;
          }
        }
      }
    }
  }
}

static void strides_of(int ndim, const int64_t* shape, int64_t* str) {
  int64_t acc = 1;
  for (int d = ndim - 1; d >= 0; --d) { str[d] = acc; acc *= shape[d]; }
}

int or_xcorr_zpad(int ndim, const double* s, const int64_t* ms, const double* k,
                  const int64_t* ns, const int64_t* pl, const int64_t* os, double* out) {
  if (ndim < 1 || ndim > OR_MAXDIM) return 1;
  int64_t sstr[OR_MAXDIM], kstr[OR_MAXDIM];
  strides_of(ndim, ms, sstr);
  strides_of(ndim, ns, kstr);
  int64_t total = 1;
  for (int d = 0; d < ndim; ++d) total *= os[d];
  memset(out, 0, (size_t)total * sizeof(double));
  if (total == 0) return 0;
  xcorr_rows(ndim, s, ms, sstr, k, ns, kstr, pl, os, out);
  return 0;
}

/* VALID correlation = zero-pad variant with no padding (_loops.py:27-69,201-208). */
int or_xcorr_valid(int ndim, const double* s, const int64_t* ms, const double* k,
                   const int64_t* ns, double* out) {
  int64_t pl[OR_MAXDIM], os[OR_MAXDIM];
  for (int d = 0; d < ndim; ++d) {
    pl[d] = 0;
    os[d] = ms[d] - ns[d] + 1;
    if (os[d] < 1) return 2;
  }
  return or_xcorr_zpad(ndim, s, ms, k, ns, pl, os, out);
}

/* np.pad(s, pads, mode="edge") for any rank (conv.py:146-148). */
int or_pad_edge(int ndim, const double* s, const int64_t* ms, const int64_t* padl,
                const int64_t* padr, double* out) {
  int64_t ps[OR_MAXDIM], sstr[OR_MAXDIM];
  int64_t total = 1;
  for (int d = 0; d < ndim; ++d) { ps[d] = ms[d] + padl[d] + padr[d]; total *= ps[d]; }
  strides_of(ndim, ms, sstr);
  for (int64_t i = 0; i < total; ++i) {
    int64_t rem = i, off = 0;
    for (int d = ndim - 1; d >= 0; --d) {
      int64_t c = rem % ps[d];
      rem /= ps[d];
      int64_t src = c - padl[d];
      if (src < 0) src = 0;
      if (src >= ms[d]) src = ms[d] - 1;
      off += src * sstr[d];
    }
    out[i] = s[off];
  }
  return 0;
}

/* conv._direct (conv.py:133-150): shape 0=FULL 1=SAME 2=VALID, boundary
 * 0=ZERO 1=REPLICATE, flip=1 for true convolution (reflected kernel).
 * Output extents must have been computed by the caller (shape law). */
int or_direct(int ndim, const double* s, const int64_t* ms, const double* k,
              const int64_t* ns, int shape, int boundary, int flip, double* out) {
  if (ndim < 1 || ndim > OR_MAXDIM) return 1;
  int64_t kn = 1;
  for (int d = 0; d < ndim; ++d) kn *= ns[d];
  double* kr = (double*)malloc((size_t)(kn ? kn : 1) * sizeof(double));
  /* reflect(k): reverse every axis == reverse the flat row-major buffer */
  for (int64_t i = 0; i < kn; ++i) kr[i] = flip ? k[kn - 1 - i] : k[i];
  int rc = 0;
  int64_t pl[OR_MAXDIM], os[OR_MAXDIM];
  if (shape == 2) {
    rc = or_xcorr_valid(ndim, s, ms, kr, ns, out);
  } else if (shape == 0) {
    for (int d = 0; d < ndim; ++d) { pl[d] = ns[d] - 1; os[d] = ms[d] + ns[d] - 1; }
    rc = or_xcorr_zpad(ndim, s, ms, kr, ns, pl, os, out);
  } else if (boundary == 1) {
    int64_t padl[OR_MAXDIM], padr[OR_MAXDIM], ps[OR_MAXDIM];
    int64_t total = 1;
    for (int d = 0; d < ndim; ++d) {
      padl[d] = (ns[d] - 1) - (ns[d] - 1) / 2; /* _same_pads: ceil((n-1)/2) */
      padr[d] = (ns[d] - 1) / 2;
      ps[d] = ms[d] + padl[d] + padr[d];
      total *= ps[d];
    }
    double* padded = (double*)malloc((size_t)(total ? total : 1) * sizeof(double));
    or_pad_edge(ndim, s, ms, padl, padr, padded);
    rc = or_xcorr_valid(ndim, padded, ps, kr, ns, out);
    free(padded);
  } else {
    for (int d = 0; d < ndim; ++d) { pl[d] = (ns[d] - 1) - (ns[d] - 1) / 2; os[d] = ms[d]; }
    rc = or_xcorr_zpad(ndim, s, ms, kr, ns, pl, os, out);
  }
  free(kr);
  return rc;
}

/* ----------------------------------------------------------------- ttc --- */

/* numpy's pairwise summation of a contiguous double array
 * (numpy/_core/src/umath/loops_utils.h.src, DOUBLE_pairwise_sum), which is
 * what np.sum does for the contiguous product temporaries of
 * build_normal_system (ttc.py:113-120). */
static double pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
  }
}

/* derivatives_3d (ttc.py:82-91): three VALID 3-D correlations of the stacked
 * pair with the 2x2x2 quarter-weight stencils _DX/_DY/_DT (ttc.py:29-31),
 * taps in [t][y][x] row-major order. */
void or_derivatives(const double* a, const double* b, int64_t h, int64_t w, double* ex,
                    double* ey, double* et) {
  static const double DX[8] = {-0.25, 0.25, -0.25, 0.25, -0.25, 0.25, -0.25, 0.25};
  static const double DY[8] = {-0.25, -0.25, 0.25, 0.25, -0.25, -0.25, 0.25, 0.25};
  static const double DT[8] = {-0.25, -0.25, -0.25, -0.25, 0.25, 0.25, 0.25, 0.25};
  const int64_t gw = w - 1, gh = h - 1;
  for (int64_t y = 0; y < gh; ++y)
    for (int64_t x = 0; x < gw; ++x) {
      const double v[8] = {a[y * w + x],       a[y * w + x + 1], a[(y + 1) * w + x],
                           a[(y + 1) * w + x + 1], b[y * w + x],       b[y * w + x + 1],
                           b[(y + 1) * w + x],     b[(y + 1) * w + x + 1]};
      double sx = 0.0, sy = 0.0, st = 0.0;
      for (int j = 0; j < 8; ++j) {
        sx = fma(DX[j], v[j], sx);
        sy = fma(DY[j], v[j], sy);
        st = fma(DT[j], v[j], st);
      }
      ex[y * gw + x] = sx;
      ey[y * gw + x] = sy;
      et[y * gw + x] = st;
    }
}

/* radial_gradient (ttc.py:94-99): G = xc*Ex + yc*Ey, no contraction. */
void or_radial_gradient(const double* ex, const double* ey, int64_t gh, int64_t gw,
                        double* g) {
  for (int64_t y = 0; y < gh; ++y) {
    const double yc = (double)y - (double)(gh - 1) / 2.0;
    for (int64_t x = 0; x < gw; ++x) {
      const double xc = (double)x - (double)(gw - 1) / 2.0;
      const double p = xc * ex[y * gw + x];
      const double q = yc * ey[y * gw + x];
      g[y * gw + x] = p + q;
    }
  }
}

/* build_normal_system (ttc.py:102-120).  sums[11] = m00 m01 m02 m11 m12 m22,
 * rhs0 rhs1 rhs2 (already negated), et2, count.  Returns 0, or 1..3 for the
 * reference's ValueError cases (border < 1, no interior). */
int or_normal_system(const double* ex, const double* ey, const double* g, const double* et,
                     int64_t gh, int64_t gw, int64_t border, double* sums) {
  if (border < 1) return 1;
  if (gh <= 2 * border || gw <= 2 * border) return 2;
  const int64_t ih = gh - 2 * border, iw = gw - 2 * border, n = ih * iw;
  double* tmp = (double*)malloc((size_t)n * sizeof(double));
  const double* f[4] = {ex, ey, g, et};
  /* product order of ttc.py:113-120 */
  static const int pa[10] = {0, 0, 0, 1, 1, 2, 0, 1, 2, 3};
  static const int pb[10] = {0, 1, 2, 1, 2, 2, 3, 3, 3, 3};
  for (int q = 0; q < 10; ++q) {
    int64_t i = 0;
    for (int64_t y = border; y < gh - border; ++y)
      for (int64_t x = border; x < gw - border; ++x, ++i)
        tmp[i] = f[pa[q]][y * gw + x] * f[pb[q]][y * gw + x];
    double sm = pairwise_sum(tmp, n);
    sums[q] = (q >= 6 && q <= 8) ? -sm : sm;
  }
  sums[10] = (double)n;
  free(tmp);
  return 0;
}

/* _ldlt_solve + solve_ttc (ttc.py:123-184).  est[10] = a b c x0 y0 ttc
 * residual misfit level degenerate. */
void or_solve_ttc(const double* sums, double c_min, double* est) {
  const double m00 = sums[0], m01 = sums[1], m02 = sums[2], m11 = sums[3], m12 = sums[4],
               m22 = sums[5];
  const double r0 = sums[6], r1 = sums[7], r2 = sums[8], et2 = sums[9], count = sums[10];
  int degenerate = 0;
  double v0 = 0, v1 = 0, v2 = 0;
  double maxdiag = m00;
  if (m11 > maxdiag) maxdiag = m11;
  if (m22 > maxdiag) maxdiag = m22;
  if (maxdiag <= 0.0) {
    degenerate = 1;
  } else {
    const double tol = 1e-10 * maxdiag;
    const double d0 = m00;
    if (d0 < tol) {
      degenerate = 1;
    } else {
      const double l10 = m01 / d0;
      const double l20 = m02 / d0;
      const double d1 = m11 - l10 * l10 * d0;
      if (d1 < tol) {
        degenerate = 1;
      } else {
        const double l21 = (m12 - l20 * l10 * d0) / d1;
        const double d2 = m22 - l20 * l20 * d0 - l21 * l21 * d1;
        if (d2 < tol) {
          degenerate = 1;
        } else {
          const double z0 = r0;
          const double z1 = r1 - l10 * z0;
          const double z2 = r2 - l20 * z0 - l21 * z1;
          const double y0 = z0 / d0, y1 = z1 / d1, y2 = z2 / d2;
          v2 = y2;
          v1 = y1 - l21 * v2;
          v0 = y0 - l10 * v1 - l20 * v2;
        }
      }
    }
  }
  if (degenerate) {
    const double nan = NAN;
    est[0] = est[1] = est[2] = est[3] = est[4] = est[5] = nan;
    est[6] = count != 0.0 ? et2 / count : nan;
    est[7] = INFINITY;
    est[8] = 0.0;
    est[9] = 1.0;
    return;
  }
  /* v @ rhs: numpy's 3-element float64 dot is an FMA chain (measured bitwise
   * against numpy 2.3 on 20k random triples) */
  double vr = fma(v2, r2, fma(v1, r1, v0 * r0));
  double j = et2 - vr;
  if (0.0 > j) j = 0.0; /* python max(x, 0.0) keeps x unless 0.0 > x */
  est[0] = v0;
  est[1] = v1;
  est[2] = v2;
  est[6] = j / count;
  est[7] = et2 > 0.0 ? j / et2 : INFINITY;
  if (fabs(v2) < c_min) {
    est[3] = NAN;
    est[4] = NAN;
    est[5] = INFINITY;
  } else {
    est[3] = -v0 / v2;
    est[4] = -v1 / v2;
    est[5] = 1.0 / v2;
  }
  est[8] = 0.0;
  est[9] = 0.0;
}

/* downsample (ttc.py:187-204): crop to even, 2x2 block mean evaluated as
 * 0.25*(((f00+f01)+f10)+f11), then 5x5 binomial SAME with REPLICATE
 * (edge pad by 2, VALID correlation, conv.py:146-148). */
int or_downsample(const double* img, int64_t h, int64_t w, double* out) {
  if (h < 2 || w < 2) return 1;
  const int64_t dh = h / 2, dw = w / 2;
  double* dec = (double*)malloc((size_t)(dh * dw) * sizeof(double));
  for (int64_t y = 0; y < dh; ++y)
    for (int64_t x = 0; x < dw; ++x) {
      const double* r0 = img + (2 * y) * w + 2 * x;
      const double* r1 = r0 + w;
      dec[y * dw + x] = 0.25 * (((r0[0] + r0[1]) + r1[0]) + r1[1]);
    }
  static const double b[5] = {1.0 / 16.0, 4.0 / 16.0, 6.0 / 16.0, 4.0 / 16.0, 1.0 / 16.0};
  double k[25];
  for (int i = 0; i < 5; ++i)
    for (int j = 0; j < 5; ++j) k[i * 5 + j] = b[i] * b[j];
  int64_t ms[2] = {dh, dw}, ns[2] = {5, 5};
  int rc = or_direct(2, dec, ms, k, ns, /*SAME*/ 1, /*REPLICATE*/ 1, /*flip*/ 0, out);
  free(dec);
  return rc;
}

/* _estimate_at (ttc.py:215-225) on frames already at `level`. */
static void estimate_at(const double* a, const double* b, int64_t h, int64_t w, int level,
                        double c_min, double* est) {
  const int64_t gh = h - 1, gw = w - 1, n = gh * gw;
  double* buf = (double*)malloc((size_t)(4 * n) * sizeof(double));
  double *ex = buf, *ey = buf + n, *et = buf + 2 * n, *g = buf + 3 * n;
  or_derivatives(a, b, h, w, ex, ey, et);
  or_radial_gradient(ex, ey, gh, gw, g);
  double sums[11];
  or_normal_system(ex, ey, g, et, gh, gw, 1, sums);
  or_solve_ttc(sums, c_min, est);
  const double scale = ldexp(1.0, level);
  est[8] = (double)level;
  est[3] = est[3] * scale;
  est[4] = est[4] * scale;
  free(buf);
}

/* estimate_fixed (ttc.py:228-245).  Returns 1 for level < 0, 2 for extents
 * below 4 after `level` halvings. */
int or_estimate_fixed(const double* a, const double* b, int64_t h, int64_t w, int level,
                      double c_min, double* est) {
  if (level < 0) return 1;
  int64_t lh = h, lw = w;
  for (int i = 0; i < level; ++i) { lh /= 2; lw /= 2; }
  if (lh < 4 || lw < 4) return 2;
  double* cur = (double*)malloc((size_t)(2 * h * w) * sizeof(double));
  double* nxt = (double*)malloc((size_t)(2 * h * w) * sizeof(double));
  memcpy(cur, a, (size_t)(h * w) * sizeof(double));
  memcpy(cur + h * w, b, (size_t)(h * w) * sizeof(double));
  int64_t ch = h, cw = w;
  for (int i = 0; i < level; ++i) {
    or_downsample(cur, ch, cw, nxt);
    or_downsample(cur + ch * cw, ch, cw, nxt + (ch / 2) * (cw / 2));
    ch /= 2;
    cw /= 2;
    double* t = cur; cur = nxt; nxt = t;
  }
  estimate_at(cur, cur + ch * cw, ch, cw, level, c_min, est);
  free(cur);
  free(nxt);
  return 0;
}

/* estimate_multiscale (ttc.py:248-279).  est[8] = -1 encodes the reference's
 * `None` result (frames smaller than 4 at level 0). */
int or_estimate_multiscale(const double* a, const double* b, int64_t h, int64_t w,
                           int max_level, double c_min, double* est) {
  if (max_level < 0) return 1;
  double* cur = (double*)malloc((size_t)(2 * h * w + 2) * sizeof(double));
  double* nxt = (double*)malloc((size_t)(2 * h * w + 2) * sizeof(double));
  memcpy(cur, a, (size_t)(h * w) * sizeof(double));
  memcpy(cur + h * w, b, (size_t)(h * w) * sizeof(double));
  int64_t ch = h, cw = w;
  int have_best = 0;
  double best[10], prev_misfit = 0.0, e[10];
  int have_prev = 0;
  for (int level = 0; level <= max_level; ++level) {
    if ((ch < cw ? ch : cw) < 4) break;
    estimate_at(cur, cur + ch * cw, ch, cw, level, c_min, e);
    if (!have_best || e[7] < best[7]) { memcpy(best, e, sizeof(best)); have_best = 1; }
    if (have_prev && !(e[7] < prev_misfit * (1.0 - 1e-3))) break;
    prev_misfit = e[7];
    have_prev = 1;
    if (level < max_level && ((ch / 2) < (cw / 2) ? (ch / 2) : (cw / 2)) >= 4) {
      or_downsample(cur, ch, cw, nxt);
      or_downsample(cur + ch * cw, ch, cw, nxt + (ch / 2) * (cw / 2));
      ch /= 2;
      cw /= 2;
      double* t = cur; cur = nxt; nxt = t;
    } else {
      break;
    }
  }
  free(cur);
  free(nxt);
  if (!have_best) {
    for (int i = 0; i < 10; ++i) est[i] = NAN;
    est[8] = -1.0;
    return 0;
  }
  memcpy(est, best, sizeof(best));
  return 0;
}

/* run_sequence (ttc.py:282-305): row i from frames (i, i+1); max_level < 0
 * selects the fixed-level path.  Pairs are independent, so the loop is
 * spread over `nthreads` OpenMP threads (0 = all); each row's arithmetic is
 * unchanged by the thread count. */
int or_run_sequence(const double* frames, int64_t n, int64_t h, int64_t w, int level,
                    int max_level, double c_min, double* est, int nthreads) {
  if (n < 2) return 1;
  if (max_level < 0) {
    int64_t lh = h, lw = w;
    for (int i = 0; i < level; ++i) { lh /= 2; lw /= 2; }
    if (level < 0) return 2;
    if (lh < 4 || lw < 4) return 3;
  }
  int rc_any = 0;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(| : rc_any)
#endif
  for (int64_t i = 0; i < n - 1; ++i) {
    const double* a = frames + i * h * w;
    const double* b = a + h * w;
    int rc = max_level >= 0 ? or_estimate_multiscale(a, b, h, w, max_level, c_min, est + i * 10)
                            : or_estimate_fixed(a, b, h, w, level, c_min, est + i * 10);
    rc_any |= rc;
  }
  (void)nthreads;
  return rc_any;
}

/* Batch of independent `direct` calls over `nb` signals sharing one kernel
 * (cfg1 CPU baseline); spread over OpenMP threads. */
int or_direct_batch(int ndim, const double* s, const int64_t* ms, int64_t nb, const double* k,
                    const int64_t* ns, int shape, int boundary, int flip, double* out,
                    int64_t out_elems, int nthreads) {
  int64_t sn = 1;
  for (int d = 0; d < ndim; ++d) sn *= ms[d];
  int rc_any = 0;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(| : rc_any)
#endif
  for (int64_t i = 0; i < nb; ++i)
    rc_any |= or_direct(ndim, s + i * sn, ms, k, ns, shape, boundary, flip, out + i * out_elems);
  (void)nthreads;
  return rc_any;
}

int or_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
