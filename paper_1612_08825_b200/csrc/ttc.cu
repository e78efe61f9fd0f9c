// Time-to-contact hot path (K5-K7) for sm_100a.
//
// Reference (paths under /root/reference/pkg/src/convtact):
//   derivatives_3d      ttc.py:82-91   (2x2x2 quarter-weight stencils ttc.py:28-31)
//   radial_gradient     ttc.py:94-99
//   build_normal_system ttc.py:102-120
//   _ldlt_solve / solve_ttc  ttc.py:123-184
//   downsample          ttc.py:187-204
//   _estimate_at / estimate_fixed / estimate_multiscale / run_sequence  ttc.py:207-305
//
// The fused kernel (ttc_moments_kernel) is the product's hot loop: one CTA
// owns a band of BR grid rows x 255 grid columns of one video and walks a
// chunk of consecutive frames.  Frame bands arrive by TMA into a 3-deep ring
// of shared-memory buffers (mbarrier-tracked), so every frame is read from
// HBM once per band and the two frames of pair t are both resident; no
// derivative field is ever written.  Per pixel it evaluates the cube
// stencils from time sums P = a + b and differences D = b - a (4x-scaled:
// Ex' = dP_y + dP_y+1, Ey' = hP_y+1 - hP_y, Et' = sD_y + sD_y+1), and
// accumulates per-column moments with G folded out algebraically
// (G = xc*Ex + yc*Ey; with H = yc*Ey the G moments are xc-weighted column
// sums plus sums of Ex*H, Ey*H, H*Et, H*H).  Per pair the CTA reduces its
// ten sums (warp shuffle, then shared memory) into a per-band partial; a
// second kernel adds the partials in a fixed order, so results do not depend
// on scheduling (bit-reproducible run to run and across shard counts).
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "moments.cuh"
#include "tma.cuh"

namespace ct {
namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------ fields ------

template <typename T>
__device__ __forceinline__ T fmx(T a, T b, T c);
template <>
__device__ __forceinline__ double fmx(double a, double b, double c) {
  return fma(a, b, c);
}
template <>
__device__ __forceinline__ float fmx(float a, float b, float c) {
  return fmaf(a, b, c);
}

// derivatives_3d: VALID 3-D correlation of the stacked pair with _DX/_DY/_DT,
// taps in [t][y][x] order accumulated with FMA from 0 (bit-identical to the
// reference in float64).
template <typename T>
__global__ void deriv_fields_kernel(const T* __restrict__ f0, const T* __restrict__ f1, int h, int w,
                                    T* ex, T* ey, T* et) {
  const int gw = w - 1, gh = h - 1;
  const int64_t n = (int64_t)gh * gw;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / gw), x = (int)(i - (int64_t)y * gw);
    const T v[8] = {f0[(int64_t)y * w + x], f0[(int64_t)y * w + x + 1], f0[(int64_t)(y + 1) * w + x],
                    f0[(int64_t)(y + 1) * w + x + 1], f1[(int64_t)y * w + x], f1[(int64_t)y * w + x + 1],
                    f1[(int64_t)(y + 1) * w + x], f1[(int64_t)(y + 1) * w + x + 1]};
    const T q = T(0.25), m = T(-0.25);
    T sx = T(0), sy = T(0), st = T(0);
    const T kx[8] = {m, q, m, q, m, q, m, q};
    const T ky[8] = {m, m, q, q, m, m, q, q};
    const T kt[8] = {m, m, m, m, q, q, q, q};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sx = fmx(kx[j], v[j], sx);
      sy = fmx(ky[j], v[j], sy);
      st = fmx(kt[j], v[j], st);
    }
    ex[i] = sx;
    ey[i] = sy;
    et[i] = st;
  }
}

template <typename T>
__global__ void radial_gradient_kernel(const T* __restrict__ ex, const T* __restrict__ ey, int gh, int gw,
                                       T* g) {
  const int64_t n = (int64_t)gh * gw;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / gw), x = (int)(i - (int64_t)y * gw);
    // xc[None,:]*ex + yc[:,None]*ey, evaluated op by op like numpy (ttc.py:97-99)
    const double xc = (double)x - (double)(gw - 1) / 2.0;
    const double yc = (double)y - (double)(gh - 1) / 2.0;
    const double pr = __dmul_rn(xc, (double)ex[i]);
    const double qr = __dmul_rn(yc, (double)ey[i]);
    g[i] = (T)__dadd_rn(pr, qr);
  }
}

constexpr int kNsBlocks = 296;
constexpr int kNsThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kNsThreads) normal_system_kernel(const T* ex, const T* ey, const T* g,
                                                                   const T* et, int gh, int gw, int border,
                                                                   double* partials) {
  const int iw = gw - 2 * border, ih = gh - 2 * border;
  const int64_t n = (int64_t)iw * ih;
  double acc[10];
#pragma unroll
  for (int q = 0; q < 10; ++q) acc[q] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / iw) + border, x = (int)(i % iw) + border;
    const int64_t o = (int64_t)y * gw + x;
    const double vx = ex[o], vy = ey[o], vg = g[o], vt = et[o];
    acc[0] += vx * vx;
    acc[1] += vx * vy;
    acc[2] += vx * vg;
    acc[3] += vy * vy;
    acc[4] += vy * vg;
    acc[5] += vg * vg;
    acc[6] += vx * vt;
    acc[7] += vy * vt;
    acc[8] += vg * vt;
    acc[9] += vt * vt;
  }
  __shared__ double red[kNsThreads / 32][10];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 10; ++q) {
    const double s = warp_sum(acc[q]);
    if (lane == 0) red[warp][q] = s;
  }
  __syncthreads();
  if (threadIdx.x < 10) {
    double s = 0.0;
    for (int w2 = 0; w2 < kNsThreads / 32; ++w2) s += red[w2][threadIdx.x];
    partials[blockIdx.x * 10 + threadIdx.x] = (threadIdx.x >= 6 && threadIdx.x <= 8) ? -s : s;
  }
}

// ------------------------------------------------------------- solve ------

// _ldlt_solve + solve_ttc (ttc.py:123-184) and the FOE scaling of
// _estimate_at (ttc.py:219-225).  Evaluated op by op (no contraction) like
// the reference's float64 scalar code; v @ rhs is numpy's FMA-chain dot.
__device__ void solve_one(const double* sm, double c_min, int level, double* e) {
  const double m00 = sm[0], m01 = sm[1], m02 = sm[2], m11 = sm[3], m12 = sm[4], m22 = sm[5];
  const double r0 = sm[6], r1 = sm[7], r2 = sm[8], et2 = sm[9], count = sm[10];
  double maxdiag = m00;
  if (m11 > maxdiag) maxdiag = m11;
  if (m22 > maxdiag) maxdiag = m22;
  bool degenerate = false;
  double v0 = 0.0, v1 = 0.0, v2 = 0.0;
  if (maxdiag <= 0.0) {
    degenerate = true;
  } else {
    const double tol = __dmul_rn(1e-10, maxdiag);
    const double d0 = m00;
    if (d0 < tol) {
      degenerate = true;
    } else {
      const double l10 = __ddiv_rn(m01, d0);
      const double l20 = __ddiv_rn(m02, d0);
      const double d1 = __dsub_rn(m11, __dmul_rn(__dmul_rn(l10, l10), d0));
      if (d1 < tol) {
        degenerate = true;
      } else {
        const double l21 = __ddiv_rn(__dsub_rn(m12, __dmul_rn(__dmul_rn(l20, l10), d0)), d1);
        const double d2 = __dsub_rn(__dsub_rn(m22, __dmul_rn(__dmul_rn(l20, l20), d0)),
                                    __dmul_rn(__dmul_rn(l21, l21), d1));
        if (d2 < tol) {
          degenerate = true;
        } else {
          const double z0 = r0;
          const double z1 = __dsub_rn(r1, __dmul_rn(l10, z0));
          const double z2 = __dsub_rn(__dsub_rn(r2, __dmul_rn(l20, z0)), __dmul_rn(l21, z1));
          const double y0 = __ddiv_rn(z0, d0), y1 = __ddiv_rn(z1, d1), y2 = __ddiv_rn(z2, d2);
          v2 = y2;
          v1 = __dsub_rn(y1, __dmul_rn(l21, v2));
          v0 = __dsub_rn(__dsub_rn(y0, __dmul_rn(l10, v1)), __dmul_rn(l20, v2));
        }
      }
    }
  }
  const double scale = ldexp(1.0, level);
  if (degenerate) {
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    e[0] = e[1] = e[2] = e[3] = e[4] = e[5] = nan;
    e[6] = count != 0.0 ? __ddiv_rn(et2, count) : nan;
    e[7] = __longlong_as_double(0x7ff0000000000000ll);
    e[8] = (double)level;
    e[9] = 1.0;
    return;
  }
  const double vr = fma(v2, r2, fma(v1, r1, __dmul_rn(v0, r0)));
  double j = __dsub_rn(et2, vr);
  if (0.0 > j) j = 0.0;
  e[0] = v0;
  e[1] = v1;
  e[2] = v2;
  e[6] = __ddiv_rn(j, count);
  e[7] = et2 > 0.0 ? __ddiv_rn(j, et2) : __longlong_as_double(0x7ff0000000000000ll);
  if (fabs(v2) < c_min) {
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    e[3] = nan;
    e[4] = nan;
    e[5] = __longlong_as_double(0x7ff0000000000000ll);
  } else {
    e[3] = __dmul_rn(__ddiv_rn(-v0, v2), scale);
    e[4] = __dmul_rn(__ddiv_rn(-v1, v2), scale);
    e[5] = __ddiv_rn(1.0, v2);
  }
  e[8] = (double)level;
  e[9] = 0.0;
}

__global__ void ttc_solve_kernel(const double* sums, int64_t count, double c_min, int level, double* est,
                                 int64_t est_stride) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  solve_one(sums + i * 11, c_min, level, est + i * est_stride);
}

// estimate_multiscale's greedy walk (ttc.py:264-279) over levels computed
// up front; identical selection because level l is only visited when every
// earlier level improved.
__global__ void multiscale_select_kernel(const double* est_levels, int64_t count, int n_levels, double* best) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const double* e = est_levels + i * n_levels * 10;
  double* o = best + i * 10;
  if (n_levels <= 0) {
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    for (int q = 0; q < 10; ++q) o[q] = nan;
    o[8] = -1.0;
    return;
  }
  int b = 0;
  double prev = 0.0;
  for (int l = 0; l < n_levels; ++l) {
    const double mf = e[l * 10 + 7];
    if (l > 0 && mf < e[b * 10 + 7]) b = l;
    if (l > 0 && !(mf < prev * (1.0 - 1e-3))) break;
    prev = mf;
  }
  for (int q = 0; q < 10; ++q) o[q] = e[b * 10 + q];
}

// ------------------------------------------------------------- pyramid ----

constexpr int kPyTileY = 32, kPyTileX = 64;  // outputs per CTA

template <typename T>
struct Vec2;
template <>
struct Vec2<double> {
  using type = double2;
};
template <>
struct Vec2<float> {
  using type = float2;
};

// downsample (ttc.py:187-204): dec = 0.25*(((f00+f01)+f10)+f11) on the even
// crop, then the 5x5 binomial over the edge-padded dec, taps row-major with
// FMA (bit-identical to the reference in float64).  A CTA stages the
// (32+4) x (64+4) dec tile (edge-clamped) in shared memory, reading each input
// pixel pair as one 2-element vector when the row pitch allows (VEC).
// DEC=false is the blur-only stage: `in` already holds the decimated images
// (dh x dw, written by the fused moments kernel), h x w are the undecimated
// extents they came from.
template <typename T, bool VEC, bool DEC = true>
__global__ void __launch_bounds__(256) pyramid_down_kernel(const T* __restrict__ in, int64_t n_images, int h,
                                                           int w, T* __restrict__ out) {
  constexpr int SY = kPyTileY + 4, SX = kPyTileX + 4;
  __shared__ T dec[SY][SX + 1];
  const int dh = h / 2, dw = w / 2;
  const int tiles_x = (dw + kPyTileX - 1) / kPyTileX;
  const int ty0 = (blockIdx.x / tiles_x) * kPyTileY, tx0 = (blockIdx.x % tiles_x) * kPyTileX;
  const T b5[5] = {T(1.0 / 16.0), T(4.0 / 16.0), T(6.0 / 16.0), T(4.0 / 16.0), T(1.0 / 16.0)};
  using V2 = typename Vec2<T>::type;
  for (int64_t img = blockIdx.y; img < n_images; img += gridDim.y) {
    const T* src = in + img * (DEC ? (int64_t)h * w : (int64_t)dh * dw);
    __syncthreads();
    if (!DEC) {  // blur-only: one warp per tile row, coalesced clamped loads, no index division
      const int lane = threadIdx.x & 31;
      for (int r = threadIdx.x >> 5; r < SY; r += blockDim.x >> 5) {
        const T* srow = src + (int64_t)min(max(ty0 + r - 2, 0), dh - 1) * dw;
#pragma unroll
        for (int c = lane; c < SX; c += 32) dec[r][c] = srow[min(max(tx0 + c - 2, 0), dw - 1)];
      }
      __syncthreads();
      // separable binomial (5 + 5 taps): this internal pyramid stage feeds the
      // multiscale search only; the public downsample keeps the reference's
      // 25-tap order (DEC=true path)
      __shared__ T hrow[SY][kPyTileX + 1];
      for (int idx = threadIdx.x; idx < SY * kPyTileX; idx += blockDim.x) {
        const int r = idx / kPyTileX, c = idx - r * kPyTileX;
        T acc = T(0);
#pragma unroll
        for (int j1 = 0; j1 < 5; ++j1) acc = fmx(b5[j1], dec[r][c + j1], acc);
        hrow[r][c] = acc;
      }
      __syncthreads();
      T* dst = out + img * (int64_t)dh * dw;
      for (int idx = threadIdx.x; idx < kPyTileY * kPyTileX; idx += blockDim.x) {
        const int r = idx / kPyTileX, c = idx - r * kPyTileX;
        const int y = ty0 + r, x = tx0 + c;
        if (y >= dh || x >= dw) continue;
        T acc = T(0);
#pragma unroll
        for (int j0 = 0; j0 < 5; ++j0) acc = fmx(b5[j0], hrow[r + j0][c], acc);
        dst[(int64_t)y * dw + x] = acc;
      }
      __syncthreads();  // hrow/dec reused by the next image of this CTA
      continue;
    }
    for (int idx = threadIdx.x; idx < SY * SX; idx += blockDim.x) {
      const int r = idx / SX, c = idx - r * SX;
      const int yy = min(max(ty0 + r - 2, 0), dh - 1), xx = min(max(tx0 + c - 2, 0), dw - 1);
      if (!DEC) {
        dec[r][c] = src[(int64_t)yy * dw + xx];
        continue;
      }
      const T* p0 = src + (int64_t)(2 * yy) * w + 2 * xx;
      const T* p1 = p0 + w;
      T f00, f01, f10, f11;
      if (VEC) {
        const V2 u = *reinterpret_cast<const V2*>(p0), l = *reinterpret_cast<const V2*>(p1);
        f00 = u.x; f01 = u.y; f10 = l.x; f11 = l.y;
      } else {
        f00 = p0[0]; f01 = p0[1]; f10 = p1[0]; f11 = p1[1];
      }
      T s;
      if constexpr (sizeof(T) == 8) {
        s = __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dadd_rn(f00, f01), f10), f11));
      } else {
        s = __fmul_rn(0.25f, __fadd_rn(__fadd_rn(__fadd_rn(f00, f01), f10), f11));
      }
      dec[r][c] = s;
    }
    __syncthreads();
    T* dst = out + img * (int64_t)dh * dw;
    for (int idx = threadIdx.x; idx < kPyTileY * kPyTileX; idx += blockDim.x) {
      const int r = idx / kPyTileX, c = idx - r * kPyTileX;
      const int y = ty0 + r, x = tx0 + c;
      if (y >= dh || x >= dw) continue;
      T acc = T(0);
#pragma unroll
      for (int j0 = 0; j0 < 5; ++j0)
#pragma unroll
        for (int j1 = 0; j1 < 5; ++j1) acc = fmx(b5[j0] * b5[j1], dec[r + j0][c + j1], acc);
      dst[(int64_t)y * dw + x] = acc;
    }
  }
}

template <typename T>
int launch_pyramid(const T* in, int64_t n_images, int h, int w, T* out, cudaStream_t st) {
  const int dh = h / 2, dw = w / 2;
  if (n_images == 0 || dh == 0 || dw == 0) return CT_OK;
  const int tiles = ((dh + kPyTileY - 1) / kPyTileY) * ((dw + kPyTileX - 1) / kPyTileX);
  dim3 grid((unsigned)tiles, (unsigned)std::min<int64_t>(n_images, 65535));
  const bool vec = (w % 2 == 0) && (reinterpret_cast<uintptr_t>(in) % (2 * sizeof(T)) == 0);
  if (vec)
    pyramid_down_kernel<T, true><<<grid, 256, 0, st>>>(in, n_images, h, w, out);
  else
    pyramid_down_kernel<T, false><<<grid, 256, 0, st>>>(in, n_images, h, w, out);
  return check_launch("pyramid_down");
}

// Blur-only pyramid stage, register sliding window: a warp owns 32 x VX
// consecutive columns (one 16-byte vector per lane) of a strip of rows of one
// decimated image and walks down it; per input row the lane's horizontal
// 5-tap sums come from its vector plus two neighbours on each side (warp
// shuffles, direct clamped loads at the warp and image edges), the last five
// horizontal rows stay in registers and each output row is their vertical
// 5-tap sum.  Same tap order and FMA chains as the shared-memory version
// (horizontal j1 = 0..4 then vertical j0 = 0..4), so results are identical.

template <typename T>
__global__ void __launch_bounds__(256) blur5_rows_kernel(const T* __restrict__ in, int64_t n_images, int dh, int dw,
                                                         int strip, T* __restrict__ out) {
  constexpr int VX = 16 / sizeof(T);
  using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  const T b5[5] = {T(1.0 / 16.0), T(4.0 / 16.0), T(6.0 / 16.0), T(4.0 / 16.0), T(1.0 / 16.0)};
  const int lane = threadIdx.x & 31;
  const int warps_x = (dw + 32 * VX - 1) / (32 * VX);
  const int n_strips = (dh + strip - 1) / strip;
  const int64_t total = n_images * n_strips * warps_x;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); item < total; item += wstride) {
    const int wx = (int)(item % warps_x);
    const int64_t t = item / warps_x;
    const int si = (int)(t % n_strips);
    const int64_t img = t / n_strips;
    const int x = (wx * 32 + lane) * VX;
    const bool valid = x < dw;
    const int y0 = si * strip, y1 = min(dh, y0 + strip);
    const T* src = in + img * (int64_t)dh * dw;
    T* dst = out + img * (int64_t)dh * dw;
    T h[5][VX];
    // row fetch (vector + the direct edge loads of lanes 0 / 31), software
    // pipelined one row ahead so the load latency overlaps the previous row
    // (measured: three rows ahead is slower)
    struct Row {
      V q;
      T e0, e1, e2, e3;
    };
    auto fetch = [&](int yy) {
      Row r;
      const T* srow = src + (int64_t)min(max(yy, 0), dh - 1) * dw;
      r.q = valid ? *reinterpret_cast<const V*>(srow + x) : V{};
      r.e0 = r.e1 = r.e2 = r.e3 = T(0);
      if (valid && lane == 0 && x > 0) {
        r.e0 = srow[x - 2];
        r.e1 = srow[x - 1];
      }
      if (valid && lane == 31 && x + VX < dw) {
        r.e2 = srow[x + VX];
        r.e3 = srow[min(x + VX + 1, dw - 1)];
      }
      return r;
    };
    Row nxt = fetch(y0 - 2);
    for (int yy = y0 - 2; yy < y1 + 2; ++yy) {
      const Row cur = nxt;
      if (yy + 1 < y1 + 2) nxt = fetch(yy + 1);
      T m[VX + 4];  // columns x-2 .. x+VX+1
      const T* qv = reinterpret_cast<const T*>(&cur.q);
#pragma unroll
      for (int c = 0; c < VX; ++c) m[c + 2] = qv[c];
      m[0] = __shfl_up_sync(0xffffffffu, qv[VX - 2], 1);
      m[1] = __shfl_up_sync(0xffffffffu, qv[VX - 1], 1);
      m[VX + 2] = __shfl_down_sync(0xffffffffu, qv[0], 1);
      m[VX + 3] = __shfl_down_sync(0xffffffffu, qv[1], 1);
      if (valid) {
        if (x == 0) {
          m[0] = m[1] = qv[0];
        } else if (lane == 0) {
          m[0] = cur.e0;
          m[1] = cur.e1;
        }
        if (x + VX >= dw) {
          m[VX + 2] = m[VX + 3] = qv[VX - 1];
        } else if (lane == 31) {
          m[VX + 2] = cur.e2;
          m[VX + 3] = cur.e3;
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int c = 0; c < VX; ++c) h[k][c] = h[k + 1][c];
#pragma unroll
      for (int c = 0; c < VX; ++c) {
        T acc = T(0);
#pragma unroll
        for (int j1 = 0; j1 < 5; ++j1) acc = fmx(b5[j1], m[c + j1], acc);
        h[4][c] = acc;
      }
      if (yy >= y0 + 2 && valid) {
        V o;
        T* ov = reinterpret_cast<T*>(&o);
#pragma unroll
        for (int c = 0; c < VX; ++c) {
          T acc = T(0);
#pragma unroll
          for (int j0 = 0; j0 < 5; ++j0) acc = fmx(b5[j0], h[j0][c], acc);
          ov[c] = acc;
        }
        *reinterpret_cast<V*>(dst + (int64_t)(yy - 2) * dw + x) = o;
      }
    }
  }
}

// TMA-fed variant of blur5_rows_kernel: every warp streams its 32 x VX column
// slab (plus 4 columns each side) through its own ring of RCH-row TMA boxes
// (own mbarriers, no CTA-wide barriers), so many rows are in flight per SM
// without registers; a lane reads its window (x-2 .. x+VX+1) from shared
// memory.  REPLICATE clamping: rows outside the image reuse the nearest
// image row's horizontal sums, columns outside take the edge value.  Same
// FMA chains as blur5_rows_kernel (bit-identical).
// ring of 3 stages x 8 rows per warp, 4 warps per CTA: cfg5 levels 1-3 blur
// 171 -> 160 us per 128-frame video against 4 x 4 rows / 8 warps (profiles/r01_moments_probe.md)
#ifndef CT_BLUR_RCH
#define CT_BLUR_RCH 8
#endif
#ifndef CT_BLUR_STAGES
#define CT_BLUR_STAGES 3
#endif
#ifndef CT_BLUR_WARPS
#define CT_BLUR_WARPS 4
#endif
constexpr int kBlurRch = CT_BLUR_RCH, kBlurStages = CT_BLUR_STAGES, kBlurWarps = CT_BLUR_WARPS;

template <typename T>
__global__ void __launch_bounds__(kBlurWarps * 32) blur5_tma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                     int64_t n_images, int dh, int dw, int strip,
                                                                     T* __restrict__ out, T* __restrict__ dec_out) {
  constexpr int VX = 16 / sizeof(T);
  constexpr int SC = 32 * VX + 2 * VX;  // staged columns per row: slab + VX each side (16-byte aligned)
  constexpr int STAGE = kBlurRch * SC;  // elements per stage
  using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  extern __shared__ __align__(128) unsigned char smem_bl[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T* ring = reinterpret_cast<T*>(smem_bl) + (size_t)wid * kBlurStages * STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_bl + (size_t)kBlurWarps * kBlurStages * STAGE * sizeof(T)) +
                   wid * kBlurStages;
  const T b5[5] = {T(1.0 / 16.0), T(4.0 / 16.0), T(6.0 / 16.0), T(4.0 / 16.0), T(1.0 / 16.0)};
  if (lane == 0)
    for (int k = 0; k < kBlurStages; ++k) mbar_init(&bars[k], 1);
  __syncwarp();
  if (lane == 0) mbar_fence_init();
  __syncwarp();
  const int warps_x = (dw + 32 * VX - 1) / (32 * VX);
  const int n_strips = (dh + strip - 1) / strip;
  const int64_t total = n_images * n_strips * warps_x;
  const int64_t wstride = (int64_t)gridDim.x * kBlurWarps;
  uint32_t uses = 0;  // boxes consumed by this warp (ring stage uses % S, phase (uses / S) & 1)
  for (int64_t item = (int64_t)blockIdx.x * kBlurWarps + wid; item < total; item += wstride) {
    const int wx = (int)(item % warps_x);
    const int64_t t = item / warps_x;
    const int si = (int)(t % n_strips);
    const int64_t img = t / n_strips;
    const int x0 = wx * 32 * VX;
    const int x = x0 + lane * VX;
    const bool valid = x < dw;
    const int y0 = si * strip, y1 = min(dh, y0 + strip);
    const int rs = max(0, y0 - 2), re = min(dh, y1 + 2);  // image rows this slab reads
    const int nchunks = (re - rs + kBlurRch - 1) / kBlurRch;
    const int64_t grow0 = img * (int64_t)dh + rs;  // tensor-map row of image row rs
    auto issue = [&](int c) {
      if (lane == 0) {
        const uint32_t u = uses + c;
        const int stg = u % kBlurStages;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bars[stg], (uint32_t)(STAGE * sizeof(T)));
        tma_load_2d(ring + stg * STAGE, &tmap, &bars[stg], x0 - VX, (int)(grow0 + (int64_t)c * kBlurRch));
      }
    };
    for (int c = 0; c < kBlurStages && c < nchunks; ++c) issue(c);
    T h[5][VX];
    T hcur[VX];
    T prev[VX];     // previous output row (the even row of a 2x2 block for dec_out)
    int have = -1;  // image row whose horizontal sums are in hcur
    for (int yy = y0 - 2; yy < y1 + 2; ++yy) {
      const int r = min(max(yy, 0), dh - 1);
      if (r != have) {  // next image row of the stream (rows are visited in order)
        const int ri = r - rs, c = ri / kBlurRch;
        const uint32_t u = uses + c;
        const int stg = u % kBlurStages;
        if (ri % kBlurRch == 0) mbar_wait(&bars[stg], (u / kBlurStages) & 1);
        const T* row = ring + stg * STAGE + (ri % kBlurRch) * SC + lane * VX;  // staged col 0 = x0 - VX
        T m[3 * VX];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const V v = *reinterpret_cast<const V*>(row + q * VX);
          const T* vv = reinterpret_cast<const T*>(&v);
#pragma unroll
          for (int e = 0; e < VX; ++e) m[q * VX + e] = vv[e];
        }
        // window x-2 .. x+VX+1 = m[VX-2 .. 2VX+1]
        if (x == 0) m[VX - 2] = m[VX - 1] = m[VX];
        if (valid && x + VX >= dw) m[2 * VX] = m[2 * VX + 1] = m[2 * VX - 1];
        else if (valid && x + VX + 1 >= dw) m[2 * VX + 1] = m[2 * VX];
#pragma unroll
        for (int cc = 0; cc < VX; ++cc) {
          T acc = T(0);
#pragma unroll
          for (int j1 = 0; j1 < 5; ++j1) acc = fmx(b5[j1], m[VX - 2 + cc + j1], acc);
          hcur[cc] = acc;
        }
        have = r;
        if (ri % kBlurRch == kBlurRch - 1 || r == re - 1) {  // chunk fully read: refill its stage
          __syncwarp();
          if (c + kBlurStages < nchunks) issue(c + kBlurStages);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int cc = 0; cc < VX; ++cc) h[k][cc] = h[k + 1][cc];
#pragma unroll
      for (int cc = 0; cc < VX; ++cc) h[4][cc] = hcur[cc];
      if (yy >= y0 + 2 && valid) {
        V o;
        T* ov = reinterpret_cast<T*>(&o);
#pragma unroll
        for (int cc = 0; cc < VX; ++cc) {
          T acc = T(0);
#pragma unroll
          for (int j0 = 0; j0 < 5; ++j0) acc = fmx(b5[j0], h[j0][cc], acc);
          ov[cc] = acc;
        }
        *reinterpret_cast<V*>(out + (img * (int64_t)dh + (yy - 2)) * dw + x) = o;
        // next level's 2x2 block means (ttc.py:202-203 on this level's even
        // crop), same add order as write_dec: ((p00 + p01) + p10) + p11
        const int y = yy - 2, ddh = dh >> 1, ddw = dw >> 1;
        if (dec_out != nullptr && (y & 1) && (y >> 1) < ddh) {
#pragma unroll
          for (int k = 0; k < VX / 2; ++k) {
            const int xd = (x >> 1) + k;
            if (xd < ddw) {
              T d;
              if constexpr (sizeof(T) == 8)
                d = __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dadd_rn(prev[2 * k], prev[2 * k + 1]), ov[2 * k]), ov[2 * k + 1]));
              else
                d = __fmul_rn(0.25f, __fadd_rn(__fadd_rn(__fadd_rn(prev[2 * k], prev[2 * k + 1]), ov[2 * k]), ov[2 * k + 1]));
              dec_out[(img * (int64_t)ddh + (y >> 1)) * ddw + xd] = d;
            }
          }
        }
#pragma unroll
        for (int cc = 0; cc < VX; ++cc) prev[cc] = ov[cc];
      }
    }
    uses += nchunks;
    __syncwarp();
  }
}

// Second half of downsample: 5x5 binomial SAME/REPLICATE over already
// decimated images (dh x dw each, from the fused moments kernel).
// 2x2 block means of n_images h x w images (the first half of downsample,
// ttc.py:202-203), for the blur fallbacks that do not emit them.
template <typename T>
__global__ void decimate_kernel(const T* __restrict__ in, int64_t n_images, int h, int w, T* __restrict__ out) {
  const int dh = h / 2, dw = w / 2;
  const int64_t n = n_images * dh * dw;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int xd = (int)(i % dw);
    const int64_t t = i / dw;
    const int yd = (int)(t % dh);
    const int64_t img = t / dh;
    const T* p0 = in + (img * h + 2 * yd) * (int64_t)w + 2 * xd;
    const T* p1 = p0 + w;
    if constexpr (sizeof(T) == 8)
      out[i] = __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dadd_rn(p0[0], p0[1]), p1[0]), p1[1]));
    else
      out[i] = __fmul_rn(0.25f, __fadd_rn(__fadd_rn(__fadd_rn(p0[0], p0[1]), p1[0]), p1[1]));
  }
}

template <typename T>
int launch_decimate(const T* in, int64_t n_images, int h, int w, T* out, cudaStream_t st) {
  const int64_t n = n_images * (h / 2) * (w / 2);
  if (n == 0) return CT_OK;
  decimate_kernel<T><<<(unsigned)std::min<int64_t>(cdiv(n, 256), (int64_t)num_sms() * 16), 256, 0, st>>>(
      in, n_images, h, w, out);
  return check_launch("decimate");
}

// blur of the block means `dec` (images of (h/2) x (w/2)) into `out`; with
// dec_out non-null also the block means of `out` (the next level's `dec`).
template <typename T>
int launch_blur_dec(const T* dec, int64_t n_images, int h, int w, T* out, cudaStream_t st, T* dec_out = nullptr) {
  const int dh = h / 2, dw = w / 2;
  if (n_images == 0 || dh == 0 || dw == 0) return CT_OK;
  constexpr int VX = 16 / sizeof(T);
  const bool aligned = dw % VX == 0 && reinterpret_cast<uintptr_t>(dec) % 16 == 0 &&
                       reinterpret_cast<uintptr_t>(out) % 16 == 0;
  if (aligned && !getenv("CT_BLUR_SMEM") && !getenv("CT_BLUR_REGS") && n_images * dh < (1ll << 31)) {
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    constexpr int SC = 32 * VX + 2 * VX;
    if (encode_tmap_2d(&tmap, dec, sizeof(T), (uint64_t)dw, (uint64_t)(n_images * dh), SC, kBlurRch)) {
      int strip = 64;
      while (strip > 8 && n_images * cdiv(dh, strip) * cdiv(dw, 32 * VX) < (int64_t)num_sms() * 24) strip /= 2;
      const int64_t items = n_images * cdiv(dh, strip) * cdiv(dw, 32 * VX);
      const size_t smem = (size_t)kBlurWarps * kBlurStages * kBlurRch * SC * sizeof(T) +
                          kBlurWarps * kBlurStages * sizeof(uint64_t);
      auto kern = blur5_tma_kernel<T>;
      CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int per_sm = 1;
      CT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlurWarps * 32, smem));
      const int64_t blocks = std::min<int64_t>(cdiv(items, kBlurWarps), (int64_t)num_sms() * std::max(1, per_sm));
      kern<<<(unsigned)blocks, kBlurWarps * 32, smem, st>>>(tmap, n_images, dh, dw, strip, out, dec_out);
      return check_launch("pyramid_blur_tma");
    }
  }
  if (aligned && !getenv("CT_BLUR_SMEM")) {
    // row strips per warp: as long as possible (the 4 halo rows are re-read)
    // while keeping >= 16 warps per SM busy
    int strip = 64;
    while (strip > 8 && n_images * cdiv(dh, strip) * cdiv(dw, 32 * VX) < (int64_t)num_sms() * 16) strip /= 2;
    const int64_t items = n_images * cdiv(dh, strip) * cdiv(dw, 32 * VX);
    const int64_t blocks = std::min<int64_t>(cdiv(items, 8), (int64_t)num_sms() * 8 * 4);
    blur5_rows_kernel<T><<<(unsigned)blocks, 256, 0, st>>>(dec, n_images, dh, dw, strip, out);
    int rc = check_launch("pyramid_blur_rows");
    if (rc || dec_out == nullptr) return rc;
    return launch_decimate<T>(out, n_images, dh, dw, dec_out, st);
  }
  const int tiles = ((dh + kPyTileY - 1) / kPyTileY) * ((dw + kPyTileX - 1) / kPyTileX);
  dim3 grid((unsigned)tiles, (unsigned)std::min<int64_t>(n_images, 65535));
  pyramid_down_kernel<T, false, false><<<grid, 256, 0, st>>>(dec, n_images, h, w, out);
  int rc = check_launch("pyramid_blur");
  if (rc || dec_out == nullptr) return rc;
  return launch_decimate<T>(out, n_images, dh, dw, dec_out, st);
}

int launch_solve(const double* sums, int64_t count, double c_min, int level, double* est, int64_t stride,
                 cudaStream_t st) {
  if (count == 0) return CT_OK;
  ttc_solve_kernel<<<(unsigned)cdiv(count, 128), 128, 0, st>>>(sums, count, c_min, level, est, stride);
  return check_launch("ttc_solve");
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

constexpr int kMaxPyr = 32;  // pyramid levels (extents < 2^31 halve at most 31 times)

// number of pyramid levels the reference visits for frames of h x w
int ms_levels(int h, int w, int max_level) {
  if (std::min(h, w) < 4) return 0;
  int n = 1;
  int lh = h, lw = w;
  for (int l = 0; l < max_level; ++l) {
    if (std::min(lh / 2, lw / 2) < 4) break;
    lh /= 2;
    lw /= 2;
    ++n;
  }
  return n;
}

// Multiscale epilogue, one CTA of kEpiThreads per frame pair: for every level
// a fixed-order sum of the band partials (thread t adds units t, t + 128, ...,
// then a warp butterfly and the four warp sums in order), the levels' solves
// side by side on the lanes of warp 0 (solve_one), and then the greedy level
// walk of multiscale_select_kernel -- one launch instead of two per level plus one.
struct EpiLevels {
  const double* partials[kMaxPyr];
  int units[kMaxPyr];
  double count[kMaxPyr];
};
constexpr int kEpiThreads = 128;

__global__ void __launch_bounds__(kEpiThreads) ms_epilogue_kernel(const EpiLevels L, int nl, int64_t np,
                                                                  double c_min, double* est) {
  constexpr int NW = kEpiThreads / 32;
  __shared__ double red[kMaxPyr][NW][10];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int64_t pr = blockIdx.x; pr < np; pr += gridDim.x) {
    for (int l = 0; l < nl; ++l) {
      double acc[10];
#pragma unroll
      for (int q = 0; q < 10; ++q) acc[q] = 0.0;
      const int units = L.units[l];
      for (int u = tid; u < units; u += kEpiThreads) {
        const double2* r = reinterpret_cast<const double2*>(L.partials[l] + (pr * units + u) * 10);
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const double2 v = r[k];
          acc[2 * k] += v.x;
          acc[2 * k + 1] += v.y;
        }
      }
#pragma unroll
      for (int q = 0; q < 10; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
      if (lane < 10) {
        double mineq = acc[0];
#pragma unroll
        for (int q = 1; q < 10; ++q)
          if (lane == q) mineq = acc[q];
        red[l][wid][lane] = mineq;
      }
    }
    __syncthreads();
    if (wid == 0) {
      double e[10];
      if (lane < nl) {  // the levels' solves run side by side
        double sm[11];
#pragma unroll
        for (int q = 0; q < 10; ++q) {
          double t = 0.0;
#pragma unroll
          for (int w = 0; w < NW; ++w) t += red[lane][w][q];
          sm[q] = t;
        }
        sm[10] = L.count[lane];
        solve_one(sm, c_min, lane, e);
      }
      // the greedy walk over the levels (multiscale_select_kernel's loop)
      int b = 0;
      double prev = 0.0, bmf = __shfl_sync(0xffffffffu, e[7], 0);
      for (int l = 0; l < nl; ++l) {
        const double mf = __shfl_sync(0xffffffffu, e[7], l);
        if (l > 0 && mf < bmf) {
          b = l;
          bmf = mf;
        }
        if (l > 0 && !(mf < prev * (1.0 - 1e-3))) break;
        prev = mf;
      }
#pragma unroll
      for (int q = 0; q < 10; ++q) {
        const double val = __shfl_sync(0xffffffffu, e[q], b);
        if (lane == 0) est[pr * 10 + q] = val;
      }
    }
    __syncthreads();
  }
}

// Workspace layout of the multiscale pipeline (run_seq with max_level >= 0 and
// pyr_moments): levels 1..nl-1 and their block-mean inputs, then one partials
// buffer per level.
template <typename T>
struct PyrPlan {
  int nl = 0;
  int lh[kMaxPyr], lw[kMaxPyr];
  size_t level_off[kMaxPyr], dec_off[kMaxPyr], part_off[kMaxPyr];
  size_t total = 0;
  PyrPlan(int64_t nv, int nf, int h, int w, int n_levels) {
    const int dt = sizeof(T) == 8 ? CT_F64 : CT_F32;
    nl = n_levels;
    lh[0] = h;
    lw[0] = w;
    for (int l = 1; l < nl; ++l) {
      lh[l] = lh[l - 1] / 2;
      lw[l] = lw[l - 1] / 2;
      const size_t bytes = align256((size_t)nv * nf * lh[l] * lw[l] * sizeof(T));
      level_off[l] = total;
      total += bytes;
      dec_off[l] = total;
      total += bytes;
    }
    for (int l = 0; l < nl; ++l) {
      part_off[l] = total;
      total += align256(moments_workspace(dt, nv, nf, lh[l], lw[l]));
    }
  }
};

// Levels 0..nl-1 of the multiscale pyramid and their band partials: level 0's
// moments also write its 2x2 block means, each blur also writes the next
// level's block means, and levels 1.. run as one moments launch.
template <typename T>
int pyr_partials(const T* frames, int64_t nv, int nf, const PyrPlan<T>& P, char* ws, cudaStream_t st,
                 cudaEvent_t after_l0 = nullptr, cudaStream_t st_l0 = nullptr) {
  // st_l0 (optional): the level-0 pass runs there and `st` (blurs, levels 1.., later the epilogue) waits
  // for it through after_l0
  const int dt = sizeof(T) == 8 ? CT_F64 : CT_F32;
  const int nl = P.nl;
  auto level = [&](int l) { return reinterpret_cast<T*>(ws + P.level_off[l]); };
  auto dec = [&](int l) { return reinterpret_cast<T*>(ws + P.dec_off[l]); };
  auto part = [&](int l) { return reinterpret_cast<double*>(ws + P.part_off[l]); };
  MomentLevel l0{frames, P.lh[0], P.lw[0], part(0), nl > 1 ? (void*)dec(1) : nullptr};
  int rc = moments_levels_launch(dt, &l0, 1, nv, nf, 1, st_l0 ? st_l0 : st);
  if (rc) return rc;
  if (after_l0) CT_CUDA(cudaEventRecord(after_l0, st_l0 ? st_l0 : st));
  if (st_l0 && after_l0) CT_CUDA(cudaStreamWaitEvent(st, after_l0, 0));
  for (int l = 1; l < nl; ++l) {
    rc = launch_blur_dec<T>(dec(l), nv * nf, P.lh[l - 1], P.lw[l - 1], level(l), st, l + 1 < nl ? dec(l + 1) : nullptr);
    if (rc) return rc;
  }
  MomentLevel lv[kMaxPyr];
  for (int l = 1; l < nl; ++l) lv[l - 1] = MomentLevel{level(l), P.lh[l], P.lw[l], part(l), nullptr};
  for (int l = 0; l < nl - 1 && rc == 0; l += kMomentLevelsPerLaunch)
    rc = moments_levels_launch(dt, lv + l, std::min(kMomentLevelsPerLaunch, nl - 1 - l), nv, nf, 1, st);
  return rc;
}

// Multiscale pipeline over many videos: the videos are split into `parts`
// consecutive groups alternating over two streams, the second stream starting
// once the first group's level-0 pass is done, so one group's memory-bound
// blurs and small levels overlap the next group's FMA-bound level-0 pass.
// Measured on 8 x 128 frames of 1080p (tools/time_cfg5.py): 1 group 4.06 us/frame, 2 groups 3.95,
// 4 groups 3.98, 8 groups 4.11.
inline int ms_parts(int64_t nv) {
  const char* e = getenv("CT_MS_PARTS");  // read per call (tests switch it)
  const int env = e ? atoi(e) : 2;
  return (int)std::max<int64_t>(1, std::min<int64_t>(env, nv));
}

// CT_MS_SCHED: 0 = groups alternate over two equal-priority streams with a phase offset, 1 = priority pipeline
inline int ms_sched() {  // read per call (tests switch it)
  const char* e = getenv("CT_MS_SCHED");
  return e ? atoi(e) : 0;
}

template <typename T>
size_t run_seq_ws(int64_t nv, int nf, int h, int w, int level, int max_level) {
  const bool ms = max_level >= 0;
  const int64_t np = nv * (nf - 1);
  if (ms) {
    const int nl = ms_levels(h, w, max_level);
    if (nl == 0) return 0;
    const int parts = ms_parts(nv);
    if (parts > 1) return 2 * align256(PyrPlan<T>((nv + parts - 1) / parts, nf, h, w, nl).total);
    return PyrPlan<T>(nv, nf, h, w, nl).total;
  }
  const int dt = sizeof(T) == 8 ? CT_F64 : CT_F32;
  size_t total = 0;
  int lh = h, lw = w;
  for (int l = 0; l <= level; ++l) {
    if (l > 0) total += align256((size_t)nv * nf * lh * lw * sizeof(T));
    if (l == level) total += align256(moments_workspace(dt, nv, nf, lh, lw));
    lh /= 2;
    lw /= 2;
  }
  return total + align256((size_t)np * 11 * sizeof(double));
}

template <typename T>
int run_seq(const T* frames, int64_t nv, int nf, int h, int w, int level, int max_level, double c_min,
            double* est, void* ws, size_t ws_bytes, cudaStream_t st) {
  const bool ms = max_level >= 0;
  const int64_t np = nv * (nf - 1);
  if (np <= 0) return CT_OK;
  const size_t need = run_seq_ws<T>(nv, nf, h, w, level, max_level);
  CT_REQUIRE(ws != nullptr && ws_bytes >= need, "run_sequence workspace too small (%zu < %zu)", ws_bytes, need);
  const int dt = sizeof(T) == 8 ? CT_F64 : CT_F32;
  char* cur = reinterpret_cast<char*>(ws);
  if (!ms) {
    const T* src = frames;
    int lh = h, lw = w;
    for (int l = 1; l <= level; ++l) {
      T* dst = reinterpret_cast<T*>(cur);
      cur += align256((size_t)nv * nf * (lh / 2) * (lw / 2) * sizeof(T));
      int rc = launch_pyramid<T>(src, nv * nf, lh, lw, dst, st);
      if (rc) return rc;
      src = dst;
      lh /= 2;
      lw /= 2;
    }
    const size_t mom = moments_workspace(dt, nv, nf, lh, lw);
    void* mom_ws = cur;
    cur += align256(mom);
    double* sums = reinterpret_cast<double*>(cur);
    int rc = moments_launch(dt, src, nv, nf, lh, lw, 1, sums, mom_ws, mom, st);
    if (rc) return rc;
    return launch_solve(sums, np, c_min, level, est, 10, st);
  }
  const int nl = ms_levels(h, w, max_level);
  if (nl == 0) {
    multiscale_select_kernel<<<(unsigned)cdiv(np, 128), 128, 0, st>>>(nullptr, np, 0, est);
    return check_launch("multiscale_select");
  }
  CT_REQUIRE(nl <= kMaxPyr, "too many pyramid levels");
  auto pipeline = [&](const T* fr, int64_t n_vid, char* w_s, double* e, cudaStream_t s, cudaEvent_t after_l0,
                      cudaStream_t s_l0 = nullptr) -> int {
    const PyrPlan<T> P(n_vid, nf, h, w, nl);
    int rc = pyr_partials<T>(fr, n_vid, nf, P, w_s, s, after_l0, s_l0);
    if (rc) return rc;
    EpiLevels L;
    for (int l = 0; l < nl; ++l) {
      L.partials[l] = reinterpret_cast<const double*>(w_s + P.part_off[l]);
      L.units[l] = moments_units(dt, n_vid, nf, P.lh[l], P.lw[l]);
      L.count[l] = (double)(P.lh[l] - 3) * (double)(P.lw[l] - 3);
    }
    const int64_t n_p = n_vid * (nf - 1);
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(n_p, (int64_t)num_sms() * 16));
    ms_epilogue_kernel<<<blocks, kEpiThreads, 0, s>>>(L, nl, n_p, c_min, e);
    return check_launch("ms_epilogue");
  };
  const int parts = ms_parts(nv);
  if (parts == 1) return pipeline(frames, nv, cur, est, st, nullptr);
  if (ms_sched() == 1) {
    // Priority pipeline: the level-0 passes of all groups queue on a low-priority stream, everything
    // after them (blurs, levels 1.., epilogue) on a high-priority stream, group k's tail gated on its
    // level-0 pass and level-0 pass k + 2 on tail k (two workspace slots).  The block scheduler hands
    // freed CTA slots to the high-priority kernels first, so a group's memory-bound tail runs beside the
    // next group's issue-bound level-0 pass instead of after it.
    constexpr int kMaxDevP = 64, kMaxParts = 16;
    static thread_local cudaStream_t lo[kMaxDevP] = {}, hi[kMaxDevP] = {};
    static thread_local cudaEvent_t ev_l0[kMaxDevP][kMaxParts] = {}, ev_done[kMaxDevP][kMaxParts] = {};
    static thread_local cudaEvent_t ev_start[kMaxDevP] = {};
    int dev = 0;
    CT_CUDA(cudaGetDevice(&dev));
    CT_REQUIRE(dev >= 0 && dev < kMaxDevP, "device index %d out of range", dev);
    CT_REQUIRE(parts <= kMaxParts, "too many multiscale groups");
    if (lo[dev] == nullptr) {
      int least = 0, greatest = 0;
      CT_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      CT_CUDA(cudaStreamCreateWithPriority(&lo[dev], cudaStreamNonBlocking, least));
      CT_CUDA(cudaStreamCreateWithPriority(&hi[dev], cudaStreamNonBlocking, greatest));
      CT_CUDA(cudaEventCreateWithFlags(&ev_start[dev], cudaEventDisableTiming));
      for (int k = 0; k < kMaxParts; ++k) {
        CT_CUDA(cudaEventCreateWithFlags(&ev_l0[dev][k], cudaEventDisableTiming));
        CT_CUDA(cudaEventCreateWithFlags(&ev_done[dev][k], cudaEventDisableTiming));
      }
    }
    const size_t slot = align256(PyrPlan<T>((nv + parts - 1) / parts, nf, h, w, nl).total);
    const int64_t fb = (int64_t)nf * h * w;
    CT_CUDA(cudaEventRecord(ev_start[dev], st));
    CT_CUDA(cudaStreamWaitEvent(lo[dev], ev_start[dev], 0));
    CT_CUDA(cudaStreamWaitEvent(hi[dev], ev_start[dev], 0));
    int rc = CT_OK;
    for (int k = 0; k < parts && rc == CT_OK; ++k) {
      const int64_t v0 = k * nv / parts, v1 = (k + 1) * nv / parts;
      if (k >= 2) CT_CUDA(cudaStreamWaitEvent(lo[dev], ev_done[dev][k - 2], 0));  // workspace slot free again
      rc = pipeline(frames + v0 * fb, v1 - v0, cur + (k & 1) * slot, est + v0 * (nf - 1) * 10, hi[dev],
                    ev_l0[dev][k], lo[dev]);
      CT_CUDA(cudaEventRecord(ev_done[dev][k], hi[dev]));
    }
    CT_CUDA(cudaStreamWaitEvent(st, ev_done[dev][parts - 1], 0));  // hi is in order: every group is done
    return rc;
  }
  // one side stream + events per (host thread, device), created once
  constexpr int kMaxDev = 64;
  static thread_local cudaStream_t sides[kMaxDev] = {};
  static thread_local cudaEvent_t evs[kMaxDev][3] = {};
  int dev = 0;
  CT_CUDA(cudaGetDevice(&dev));
  CT_REQUIRE(dev >= 0 && dev < kMaxDev, "device index %d out of range", dev);
  if (sides[dev] == nullptr) {
    CT_CUDA(cudaStreamCreateWithFlags(&sides[dev], cudaStreamNonBlocking));
    for (auto& e : evs[dev]) CT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaStream_t ss[2] = {st, sides[dev]};
  const size_t slot = align256(PyrPlan<T>((nv + parts - 1) / parts, nf, h, w, nl).total);
  const int64_t fb = (int64_t)nf * h * w;
  CT_CUDA(cudaEventRecord(evs[dev][0], st));  // the side stream starts after prior work on `st`
  CT_CUDA(cudaStreamWaitEvent(ss[1], evs[dev][0], 0));
  int rc = CT_OK;
  for (int k = 0; k < parts && rc == CT_OK; ++k) {
    const int64_t v0 = k * nv / parts, v1 = (k + 1) * nv / parts;
    if (k == 1) CT_CUDA(cudaStreamWaitEvent(ss[1], evs[dev][1], 0));  // phase offset: after group 0's level 0
    rc = pipeline(frames + v0 * fb, v1 - v0, cur + (k & 1) * slot, est + v0 * (nf - 1) * 10, ss[k & 1],
                  k == 0 ? evs[dev][1] : nullptr);
  }
  CT_CUDA(cudaEventRecord(evs[dev][2], ss[1]));  // join
  CT_CUDA(cudaStreamWaitEvent(st, evs[dev][2], 0));
  return rc;
}

// Per-level normal-system sums of every frame pair on the multiscale pyramid
// (the `[n-1][levels][11]` entry SURVEY.md 8(b) proposes, here laid out
// [levels][n_videos][n_frames-1][11]): level l is the l-fold downsample of the
// frames (block means fused into the previous level's moments kernel, then
// the 5x5 binomial), exactly the sums run_sequence's multiscale walk solves.
template <typename T>
size_t pyr_ws(int64_t nv, int nf, int h, int w, int levels) {
  return PyrPlan<T>(nv, nf, h, w, levels).total;
}

template <typename T>
int pyr_moments(const T* frames, int64_t nv, int nf, int h, int w, int levels, double* sums, void* ws,
                size_t ws_bytes, cudaStream_t st) {
  const int64_t np = nv * (nf - 1);
  if (np <= 0) return CT_OK;
  CT_REQUIRE(levels <= kMaxPyr, "too many pyramid levels");
  const size_t need = pyr_ws<T>(nv, nf, h, w, levels);
  CT_REQUIRE(ws != nullptr && ws_bytes >= need, "pyramid_moments workspace too small (%zu < %zu)", ws_bytes, need);
  const int dt = sizeof(T) == 8 ? CT_F64 : CT_F32;
  char* cur = reinterpret_cast<char*>(ws);
  const PyrPlan<T> P(nv, nf, h, w, levels);
  int rc = pyr_partials<T>(frames, nv, nf, P, cur, st);
  if (rc) return rc;
  for (int l = 0; l < levels; ++l) {
    const double count = (double)(P.lh[l] - 3) * (double)(P.lw[l] - 3);
    rc = partials_finalize(reinterpret_cast<const double*>(cur + P.part_off[l]), np,
                           moments_units(dt, nv, nf, P.lh[l], P.lw[l]), count, sums + (size_t)l * np * 11, st);
    if (rc) return rc;
  }
  return CT_OK;
}

}  // namespace
}  // namespace ct

using namespace ct;

#define CT_DT_CHECK(dtype) CT_REQUIRE((dtype) == CT_F64 || (dtype) == CT_F32, "dtype must be CT_F64 or CT_F32")

extern "C" int ct_ttc_derivatives(int dtype, const void* first, const void* second, int64_t h, int64_t w,
                                  void* ex, void* ey, void* et, void* stream) {
  clear_error();
  CT_DT_CHECK(dtype);
  CT_REQUIRE(h >= 2 && w >= 2, "need extents >= 2 for derivatives, got (%lld, %lld)", (long long)h, (long long)w);
  CT_REQUIRE(h < (1 << 30) && w < (1 << 30), "extent too large");
  const int64_t n = (h - 1) * (w - 1);
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(n, 256), (int64_t)num_sms() * 16);
  cudaStream_t st = as_stream(stream);
  if (dtype == CT_F64)
    deriv_fields_kernel<double><<<blocks, 256, 0, st>>>((const double*)first, (const double*)second, (int)h,
                                                         (int)w, (double*)ex, (double*)ey, (double*)et);
  else
    deriv_fields_kernel<float><<<blocks, 256, 0, st>>>((const float*)first, (const float*)second, (int)h, (int)w,
                                                        (float*)ex, (float*)ey, (float*)et);
  return check_launch("derivatives");
}

extern "C" int ct_radial_gradient(int dtype, const void* ex, const void* ey, int64_t gh, int64_t gw, void* g,
                                  void* stream) {
  clear_error();
  CT_DT_CHECK(dtype);
  CT_REQUIRE(gh >= 0 && gw >= 0 && gh < (1 << 30) && gw < (1 << 30), "bad extents");
  const int64_t n = gh * gw;
  if (n == 0) return CT_OK;
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(n, 256), (int64_t)num_sms() * 16);
  cudaStream_t st = as_stream(stream);
  if (dtype == CT_F64)
    radial_gradient_kernel<double><<<blocks, 256, 0, st>>>((const double*)ex, (const double*)ey, (int)gh, (int)gw,
                                                            (double*)g);
  else
    radial_gradient_kernel<float><<<blocks, 256, 0, st>>>((const float*)ex, (const float*)ey, (int)gh, (int)gw,
                                                           (float*)g);
  return check_launch("radial_gradient");
}

extern "C" size_t ct_normal_system_workspace_bytes(int64_t gh, int64_t gw) {
  (void)gh;
  (void)gw;
  return (size_t)kNsBlocks * 10 * sizeof(double);
}

extern "C" int ct_normal_system(int dtype, const void* ex, const void* ey, const void* g, const void* et, int64_t gh,
                                int64_t gw, int64_t border, double* sums, void* workspace, size_t workspace_bytes,
                                void* stream) {
  clear_error();
  CT_DT_CHECK(dtype);
  CT_REQUIRE(border >= 1, "border must cover the derivative-kernel radius (>= 1)");
  CT_REQUIRE(gh > 2 * border && gw > 2 * border, "no interior left: grid (%lld, %lld), border %lld", (long long)gh,
             (long long)gw, (long long)border);
  CT_REQUIRE(workspace && workspace_bytes >= ct_normal_system_workspace_bytes(gh, gw), "workspace too small");
  cudaStream_t st = as_stream(stream);
  double* partials = reinterpret_cast<double*>(workspace);
  if (dtype == CT_F64)
    normal_system_kernel<double><<<kNsBlocks, kNsThreads, 0, st>>>((const double*)ex, (const double*)ey,
                                                                    (const double*)g, (const double*)et, (int)gh,
                                                                    (int)gw, (int)border, partials);
  else
    normal_system_kernel<float><<<kNsBlocks, kNsThreads, 0, st>>>((const float*)ex, (const float*)ey,
                                                                   (const float*)g, (const float*)et, (int)gh,
                                                                   (int)gw, (int)border, partials);
  int rc = check_launch("normal_system");
  if (rc) return rc;
  const double count = (double)(gh - 2 * border) * (double)(gw - 2 * border);
  return partials_finalize(partials, 1, kNsBlocks, count, sums, st);
}

extern "C" size_t ct_ttc_moments_workspace_bytes(int dtype, int64_t n_videos, int64_t n_frames, int64_t h,
                                                 int64_t w) {
  return moments_workspace(dtype, n_videos, (int)n_frames, (int)h, (int)w);
}

extern "C" int ct_ttc_moments(int dtype, const void* frames, int64_t n_videos, int64_t n_frames, int64_t h,
                              int64_t w, double* sums, void* workspace, size_t workspace_bytes, void* stream) {
  clear_error();
  CT_DT_CHECK(dtype);
  CT_REQUIRE(n_frames >= 2, "need at least two frames");
  CT_REQUIRE(h >= 4 && w >= 4, "frames of (%lld, %lld) leave no interior, need >= 4", (long long)h, (long long)w);
  CT_REQUIRE(h < (1 << 30) && w < (1 << 30) && n_frames < (1 << 30) && n_videos >= 0, "bad extents");
  return moments_launch(dtype, frames, n_videos, (int)n_frames, (int)h, (int)w, 1, sums, workspace, workspace_bytes,
                        as_stream(stream));
}

extern "C" int ct_ttc_solve(const double* sums, int64_t count, double c_min, int level, double* est, void* stream) {
  clear_error();
  CT_REQUIRE(count >= 0 && level >= 0, "bad arguments");
  return launch_solve(sums, count, c_min, level, est, 10, as_stream(stream));
}

extern "C" int ct_pyramid_down(int dtype, const void* in, int64_t n_images, int64_t h, int64_t w, void* out,
                               void* stream) {
  clear_error();
  CT_DT_CHECK(dtype);
  CT_REQUIRE(h >= 2 && w >= 2, "cannot halve extents (%lld, %lld)", (long long)h, (long long)w);
  CT_REQUIRE(h < (1 << 30) && w < (1 << 30) && n_images >= 0, "bad extents");
  cudaStream_t st = as_stream(stream);
  if (dtype == CT_F64) return launch_pyramid<double>((const double*)in, n_images, (int)h, (int)w, (double*)out, st);
  return launch_pyramid<float>((const float*)in, n_images, (int)h, (int)w, (float*)out, st);
}

extern "C" int ct_ttc_multiscale_select(const double* est_levels, int64_t count, int n_levels, double* best,
                                        void* stream) {
  clear_error();
  CT_REQUIRE(count >= 0 && n_levels >= 0, "bad arguments");
  if (count == 0) return CT_OK;
  multiscale_select_kernel<<<(unsigned)cdiv(count, 128), 128, 0, as_stream(stream)>>>(est_levels, count, n_levels,
                                                                                      best);
  return check_launch("multiscale_select");
}

// multiscale: the reference accepts any max_level (its walk stops once the
// extents drop below 4, ttc.py:264-279) and ignores `level`; extents < 2^30
// stop the walk long before kMaxPyr levels
static int clamp_max_level(int max_level) { return std::min(max_level, kMaxPyr - 1); }

extern "C" size_t ct_run_sequence_workspace_bytes(int dtype, int64_t n_videos, int64_t n_frames, int64_t h, int64_t w,
                                                  int level, int max_level) {
  if (n_frames < 2 || h < 1 || w < 1) return 0;
  max_level = clamp_max_level(max_level);
  if (dtype == CT_F64) return run_seq_ws<double>(n_videos, (int)n_frames, (int)h, (int)w, level, max_level);
  return run_seq_ws<float>(n_videos, (int)n_frames, (int)h, (int)w, level, max_level);
}

static int check_run_seq_args(int64_t n_frames, int64_t h, int64_t w, int level, int max_level) {
  CT_REQUIRE(n_frames >= 2, "need at least two frames");
  CT_REQUIRE(h < (1 << 30) && w < (1 << 30) && n_frames < (1 << 30), "extent too large");
  if (max_level < 0) {
    CT_REQUIRE(level >= 0, "level must be >= 0");
    int64_t lh = h, lw = w;
    for (int i = 0; i < level && lh >= 4 && lw >= 4; ++i) {
      lh /= 2;
      lw /= 2;
    }
    CT_REQUIRE(lh >= 4 && lw >= 4, "extents (%lld, %lld) leave (%lld, %lld) after %d halvings, need >= 4",
               (long long)h, (long long)w, (long long)lh, (long long)lw, level);
  }
  return CT_OK;
}

extern "C" int ct_run_sequence(int dtype, const void* frames, int64_t n_videos, int64_t n_frames, int64_t h,
                               int64_t w, int level, int max_level, double c_min, double* est, void* workspace,
                               size_t workspace_bytes, void* stream) {
  clear_error();
  CT_DT_CHECK(dtype);
  int rc = check_run_seq_args(n_frames, h, w, level, max_level);
  if (rc) return rc;
  max_level = clamp_max_level(max_level);
  cudaStream_t st = as_stream(stream);
  if (dtype == CT_F64)
    return run_seq<double>((const double*)frames, n_videos, (int)n_frames, (int)h, (int)w, level, max_level, c_min,
                           est, workspace, workspace_bytes, st);
  return run_seq<float>((const float*)frames, n_videos, (int)n_frames, (int)h, (int)w, level, max_level, c_min, est,
                        workspace, workspace_bytes, st);
}

static int check_pyr_args(int64_t n_frames, int64_t h, int64_t w, int levels) {
  CT_REQUIRE(n_frames >= 2, "need at least two frames");
  CT_REQUIRE(h < (1 << 30) && w < (1 << 30) && n_frames < (1 << 30), "extent too large");
  CT_REQUIRE(levels >= 1 && levels < 31, "levels must be in [1, 30]");
  int64_t lh = h, lw = w;
  for (int i = 0; i < levels - 1; ++i) {
    lh /= 2;
    lw /= 2;
  }
  CT_REQUIRE(lh >= 4 && lw >= 4, "extents (%lld, %lld) leave (%lld, %lld) after %d halvings, need >= 4",
             (long long)h, (long long)w, (long long)lh, (long long)lw, levels - 1);
  return CT_OK;
}

extern "C" size_t ct_ttc_pyramid_moments_workspace_bytes(int dtype, int64_t n_videos, int64_t n_frames, int64_t h,
                                                        int64_t w, int levels) {
  if (n_frames < 2 || h < 1 || w < 1 || levels < 1 || levels > 30) return 0;
  if (dtype == CT_F64) return pyr_ws<double>(n_videos, (int)n_frames, (int)h, (int)w, levels);
  return pyr_ws<float>(n_videos, (int)n_frames, (int)h, (int)w, levels);
}

extern "C" int ct_ttc_pyramid_moments(int dtype, const void* frames, int64_t n_videos, int64_t n_frames, int64_t h,
                                      int64_t w, int levels, double* sums, void* workspace, size_t workspace_bytes,
                                      void* stream) {
  clear_error();
  CT_DT_CHECK(dtype);
  int rc = check_pyr_args(n_frames, h, w, levels);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  if (dtype == CT_F64)
    return pyr_moments<double>((const double*)frames, n_videos, (int)n_frames, (int)h, (int)w, levels, sums,
                               workspace, workspace_bytes, st);
  return pyr_moments<float>((const float*)frames, n_videos, (int)n_frames, (int)h, (int)w, levels, sums, workspace,
                            workspace_bytes, st);
}
