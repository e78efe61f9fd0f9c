// K5: fused derivative stencils + radial gradient + normal-system moments
// over every consecutive frame pair (replaces derivatives_3d +
// radial_gradient + build_normal_system, ttc.py:82-120, inside the
// run_sequence loop ttc.py:299-304).
//
// Layout and schedule
//   * A CTA (256 threads, one grid column each; fp32: 128 threads, two
//     columns each) owns a band of BR grid rows x
//     up to 255 grid columns of one video and walks a chunk of consecutive
//     frames.  Frame bands (BR+1 rows x 256 columns) arrive by TMA into a
//     ring of NB shared-memory buffers tracked by mbarriers: while pair
//     (t-1, t) is computed from two resident buffers, frames t+1.. are in flight.
//     Every frame is read from HBM once per band (the one-row band halo is
//     shared with the neighbouring CTA through L2); no derivative field is
//     ever written.
//   * Per pixel (4x-scaled stencils, the x0.25 of ttc.py:29-31 is applied as
//     an exact x1/16 on the sums): P = a + b, D = b - a per frame column;
//     hP = P[x] + P[x+1], dP = P[x+1] - P[x], sD = D[x] + D[x+1] per row;
//     Ex' = dP_y + dP_y+1, Ey' = hP_y+1 - hP_y, Et' = sD_y + sD_y+1.
//   * G = xc*Ex + yc*Ey is folded out algebraically: with H = yc*Ey a thread
//     (fixed column, fixed xc) accumulates S = {Ex^2, ExEy, Ey^2, ExEt, EyEt,
//     Et^2} and U = {Ex H, Ey H, H Et, H H}; then sum(Ex G) = xc S1 + U1,
//     sum(Ey G) = xc S2 + U2, sum(G Et) = xc S4 + U3, sum(G^2) = xc^2 S1 +
//     2 xc U1 + U4, with the U sums accumulated under band-relative y
//     weights (see sweep()); ~20 FP64 ops per grid pixel.
//   * Per pair the 256 per-thread sums become one partial per band: in the
//     warp-streaming kernel (ttc_moments_ws_kernel, used whenever the frames
//     admit a TMA map) each warp reduces its lanes with a transpose-reduce
//     butterfly and deposits one partial; two pairs later (when the frame ring
//     guarantees every warp has deposited) one warp, rotating, adds them in a
//     fixed tree, with no CTA barrier; the CTA-barrier kernel (ttc_moments_kernel,
//     LDG loader for frames without a TMA map) reduces through shared memory
//     in a fixed tree.  moments_finalize adds the band partials in a fixed
//     order.  Results are bit-reproducible and independent of how pairs are
//     chunked or sharded.
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "moments.cuh"
#include "tma.cuh"

namespace ct {
namespace {

// BC = frame columns per tile (TMA box inner extent) = threads per CTA; a
// frame that fits one tile uses BC-1 grid columns of it.
// With several column tiles the stride is 252 grid columns: a TMA box must
// start 16-byte aligned (a start at element 255 faults with an illegal
// instruction), and 252 is a multiple of 4 f32 / 2 f64 elements.
// (multi-tile stride: BC - 4 grid columns)
#ifndef CT_MOM_TWO_COL_F32
#define CT_MOM_TWO_COL_F32 1
#endif
constexpr bool kTwoColF32 = CT_MOM_TWO_COL_F32;  // fp32: two grid columns per thread (sweep_c2)
#ifndef CT_MOM_PACKED_F32
#define CT_MOM_PACKED_F32 1
#endif
constexpr bool kPackedF32 = CT_MOM_PACKED_F32;  // fp32 interior bands use sweep_x2

template <typename T>
struct AccT {
  using type = T;  // per-thread accumulation type (f64 frames: f64; f32 frames: f32)
};

struct MomentArgs {
  const void* frames;
  double* partials;  // [n_videos][n_pairs][units][10]
  int64_t n_videos;
  int n_frames;
  int h, w, gh, gw, border;
  int n_ctiles, units;
  int chunk;      // pairs per CTA
  int use_tma;
  int tile_cols;  // grid columns per tile
  void* dec;      // optional [n_videos][n_frames][h/2][w/2]: 2x2 block means of every frame
  int dh, dw;
};

// The 2x2 block-mean decimation of downsample (ttc.py:202-203), written for
// the frame resident in `buf` while it is in shared memory, so the next
// pyramid level never re-reads the full-size frame: band rows [gy0, gy0+BR)
// and this tile's columns map to dec rows [gy0/2, (gy0+BR)/2) and dec columns
// [cx0/2, (cx0 + tile_cols + 1)/2), disjoint across CTAs.
template <typename T, int BR, int NT, int BC>
__device__ __forceinline__ void write_dec(const MomentArgs& a, const T* buf, int64_t v, int f, int gy0, int cx0,
                                          int tid) {
  constexpr int DC = BC / 2;  // dec columns per tile (at most)
  const int dy0 = gy0 >> 1, dx0 = cx0 >> 1;
  const int ndy = min(BR / 2, a.dh - dy0);
  const int ndx = min((a.tile_cols + 1) >> 1, a.dw - dx0);
  if constexpr (sizeof(T) == 4) {
    if ((a.dw & 1) == 0) {  // two dec columns per thread: one 16-byte smem read per source row, 8-byte stores
      constexpr int DC2 = DC / 2;
      static_assert(NT % DC2 == 0, "write_dec maps DC/2 dec column pairs per thread row");
      const int xp = tid % DC2;  // dec columns 2xp, 2xp + 1
      if (ndy <= 0 || 2 * xp >= ndx) return;
      const bool two = 2 * xp + 1 < ndx;
      float* dst = reinterpret_cast<float*>(a.dec) + ((v * a.n_frames + f) * (int64_t)a.dh + dy0) * a.dw + dx0 + 2 * xp;
#pragma unroll 4
      for (int yy = tid / DC2; yy < ndy; yy += NT / DC2) {
        const float4 q0 = *reinterpret_cast<const float4*>(buf + (2 * yy) * BC + 4 * xp);
        const float4 q1 = *reinterpret_cast<const float4*>(buf + (2 * yy + 1) * BC + 4 * xp);
        const float d0 = __fmul_rn(0.25f, __fadd_rn(__fadd_rn(__fadd_rn(q0.x, q0.y), q1.x), q1.y));
        const float d1 = __fmul_rn(0.25f, __fadd_rn(__fadd_rn(__fadd_rn(q0.z, q0.w), q1.z), q1.w));
        float* o = dst + (int64_t)yy * a.dw;
        if (two)
          *reinterpret_cast<float2*>(o) = make_float2(d0, d1);
        else
          o[0] = d0;
      }
      return;
    }
  }
  auto mean = [&](int yy, int xx) {
    const T* p0 = buf + (2 * yy) * BC + 2 * xx;
    const T* p1 = p0 + BC;
    if constexpr (sizeof(T) == 8)
      return __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dadd_rn(p0[0], p0[1]), p1[0]), p1[1]));
    else
      return __fmul_rn(0.25f, __fadd_rn(__fadd_rn(__fadd_rn(p0[0], p0[1]), p1[0]), p1[1]));
  };
  T* base = reinterpret_cast<T*>(a.dec) + ((v * a.n_frames + f) * (int64_t)a.dh + dy0) * a.dw + dx0;
  if constexpr (NT % DC == 0) {  // a thread keeps one dec column
    const int xx = tid % DC;
    if (ndy <= 0 || xx >= ndx) return;
#pragma unroll 4
    for (int yy = tid / DC; yy < ndy; yy += NT / DC) base[(int64_t)yy * a.dw + xx] = mean(yy, xx);
  } else {  // fewer threads than dec columns (four columns per thread)
    for (int idx = tid; idx < ndy * DC; idx += NT) {
      const int yy = idx / DC, xx = idx - yy * DC;
      if (xx < ndx) base[(int64_t)yy * a.dw + xx] = mean(yy, xx);
    }
  }
}

template <typename T, int BR, int NB, int BC, int NT = BC>
struct Smem {  // NB = frame-band buffers in the TMA ring (NB - 2 frames in flight per pair), NT threads
  static constexpr size_t buf_elems = (size_t)(BR + 1) * BC + 8;  // +8: masked right-neighbour reads
  static constexpr size_t buf_bytes = (buf_elems * sizeof(T) + 127) & ~size_t(127);
  // the reduction scratch lives in the dead previous-frame buffer; f32 bands
  // are smaller, so lane pairs are combined first (half the scratch)
  static constexpr bool half_red = buf_bytes < 10 * NT * sizeof(double);
  static constexpr int red_n = half_red ? NT / 2 : NT;
  static constexpr int seg = NT >= 256 ? 16 : NT >= 128 ? 8 : 4;  // stage-1 segments per value (10 * seg <= NT)
  static_assert(buf_bytes >= 10 * (size_t)red_n * sizeof(double), "reduction scratch must fit a band buffer");
  static constexpr size_t bars_off = NB * buf_bytes;
  static constexpr size_t part_off = bars_off + 64;
  static constexpr size_t total = part_off + 10 * seg * sizeof(double);
};

// One thread's sweep down its column of the band for one frame pair (A, B):
// m = {S1..S6, U1'..U4'} over the grid rows whose band-local frame row r lies
// in [r_beg, r_end].  The y weights are relative to the band's first grid row
// (w = r - 1), so no running coordinate is carried; the caller shifts them by
// the absolute coordinate yc0 of that row: U1 = yc0 S2 + U1', U2 = yc0 S3 +
// U2', U3 = yc0 S5 + U3', U4 = yc0^2 S3 + 2 yc0 U2' + U4'.
// The weighted sums use running sums of the running sums instead of a
// multiply per row: with K = BR rows, Q = sum_k S(k) (S after row k) is
// sum_r (K - r + 1) t_r and QQ = sum_k Q(k) is sum_r (K-r+1)(K-r+2)/2 t_r, so
//   sum_r (r-1) t_r   = K S - Q,
//   sum_r (r-1)^2 t_r = K^2 S - (2K + 1) Q + 2 QQ      (t = ey^2 for QQ);
// four adds per row replace one multiply and four FMAs.  Rows outside
// [r_beg, r_end] leave S unchanged (t_r = 0) but still advance Q and QQ.
// CHECK=false is the interior fast path (all rows, no per-row tests).
// RAW = true returns the running sums themselves in m[6..9] (Q2, Q3, Q5, QQ3);
// thread_sums<RAW> then folds the band-relative weights and the absolute
// shift into one step (three FP64 operations fewer per pair).
template <typename T, int BR, bool CHECK, int BC, bool RAW = false>
__device__ __forceinline__ void sweep(const T* __restrict__ A, const T* __restrict__ B, int col, int r_beg,
                                      int r_end, typename AccT<T>::type (&m)[10]) {
  using ACC = typename AccT<T>::type;
  ACC s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0, s6 = 0, q2 = 0, q3 = 0, q5 = 0, qq3 = 0;
  ACC hP, dP, sD;
  {
    const ACC a0 = (ACC)A[col], a1 = (ACC)A[col + 1], b0 = (ACC)B[col], b1 = (ACC)B[col + 1];
    const ACC P0 = a0 + b0, P1 = a1 + b1, D0 = b0 - a0, D1 = b1 - a1;
    hP = P0 + P1;
    dP = P1 - P0;
    sD = D0 + D1;
  }
#pragma unroll
  for (int r = 1; r <= BR; ++r) {
    const T* ra = A + r * BC + col;
    const T* rb = B + r * BC + col;
    const ACC a0 = (ACC)ra[0], a1 = (ACC)ra[1], b0 = (ACC)rb[0], b1 = (ACC)rb[1];
    const ACC P0 = a0 + b0, P1 = a1 + b1, D0 = b0 - a0, D1 = b1 - a1;
    const ACC nhP = P0 + P1, ndP = P1 - P0, nsD = D0 + D1;
    if (!CHECK || (r >= r_beg && r <= r_end)) {  // grid row gy0 + r - 1
      const ACC ex = dP + ndP;
      const ACC ey = nhP - hP;
      const ACC et = sD + nsD;
      s1 = fma(ex, ex, s1);
      s2 = fma(ex, ey, s2);
      s3 = fma(ey, ey, s3);
      s4 = fma(ex, et, s4);
      s5 = fma(ey, et, s5);
      s6 = fma(et, et, s6);
    }
    if (r == 1) {  // Q(1) = S(1), QQ(1) = Q(1)
      q2 = s2;
      q3 = s3;
      q5 = s5;
      qq3 = s3;
    } else {
      q2 += s2;
      q3 += s3;
      q5 += s5;
      qq3 += q3;
    }
    hP = nhP;
    dP = ndP;
    sD = nsD;
  }
  constexpr ACC K = ACC(BR);
  m[0] = s1; m[1] = s2; m[2] = s3; m[3] = s4; m[4] = s5; m[5] = s6;
  if constexpr (RAW) {
    m[6] = q2; m[7] = q3; m[8] = q5; m[9] = qq3;
  } else {
    m[6] = fma(K, s2, -q2);
    m[7] = fma(K, s3, -q3);
    m[8] = fma(K, s5, -q5);
    m[9] = fma(K * K, s3, fma(-(2 * K + 1), q3, 2 * qq3));
  }
}

// fp32 interior sweep with packed f32x2 arithmetic: lane .x of every pair
// register walks band rows 1..BR/2 and lane .y rows BR/2+1..BR of the same
// column, so each FADD2/FFMA2 does the work of two scalar instructions (the
// per-lane operation order is the scalar sweep's).  The two half-band sums
// are combined with the y-weight shift of the second half: with H = BR/2,
// U1 += H S2, U2 += H S3, U3 += H S5, U4 += H^2 S3 + 2 H U2 (second half).
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(*reinterpret_cast<unsigned long long*>(&a)),
      "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(*reinterpret_cast<unsigned long long*>(&a)),
      "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(*reinterpret_cast<unsigned long long*>(&a)),
      "l"(*reinterpret_cast<unsigned long long*>(&b)), "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}

template <int BR, int BC>
__device__ __forceinline__ void sweep_x2(const float* __restrict__ A, const float* __restrict__ B, int col,
                                         float (&m)[10]) {
  constexpr int H = BR / 2;
  auto ld = [&](const float* F, int r, int c) { return make_float2(F[r * BC + c], F[(r + H) * BC + c]); };
  float2 s1 = {0, 0}, s2 = {0, 0}, s3 = {0, 0}, s4 = {0, 0}, s5 = {0, 0}, s6 = {0, 0};
  float2 q2, q3, q5, qq3, hP, dP, sD;
  {
    const float2 a0 = ld(A, 0, col), a1 = ld(A, 0, col + 1), b0 = ld(B, 0, col), b1 = ld(B, 0, col + 1);
    const float2 P0 = f2add(a0, b0), P1 = f2add(a1, b1), D0 = f2sub(b0, a0), D1 = f2sub(b1, a1);
    hP = f2add(P0, P1);
    dP = f2sub(P1, P0);
    sD = f2add(D0, D1);
  }
#pragma unroll
  for (int r = 1; r <= H; ++r) {
    const float2 a0 = ld(A, r, col), a1 = ld(A, r, col + 1), b0 = ld(B, r, col), b1 = ld(B, r, col + 1);
    const float2 P0 = f2add(a0, b0), P1 = f2add(a1, b1), D0 = f2sub(b0, a0), D1 = f2sub(b1, a1);
    const float2 nhP = f2add(P0, P1), ndP = f2sub(P1, P0), nsD = f2add(D0, D1);
    const float2 ex = f2add(dP, ndP), ey = f2sub(nhP, hP), et = f2add(sD, nsD);
    s1 = f2fma(ex, ex, s1);
    s2 = f2fma(ex, ey, s2);
    s3 = f2fma(ey, ey, s3);
    s4 = f2fma(ex, et, s4);
    s5 = f2fma(ey, et, s5);
    s6 = f2fma(et, et, s6);
    if (r == 1) {
      q2 = s2;
      q3 = s3;
      q5 = s5;
      qq3 = s3;
    } else {
      q2 = f2add(q2, s2);
      q3 = f2add(q3, s3);
      q5 = f2add(q5, s5);
      qq3 = f2add(qq3, q3);
    }
    hP = nhP;
    dP = ndP;
    sD = nsD;
  }
  constexpr float K = float(H);
  // per half: U1' = K S2 - Q2, U2' = K S3 - Q3, U3' = K S5 - Q5, U4' = K^2 S3 - (2K+1) Q3 + 2 QQ3
  const float u1x = fmaf(K, s2.x, -q2.x), u1y = fmaf(K, s2.y, -q2.y);
  const float u2x = fmaf(K, s3.x, -q3.x), u2y = fmaf(K, s3.y, -q3.y);
  const float u3x = fmaf(K, s5.x, -q5.x), u3y = fmaf(K, s5.y, -q5.y);
  const float u4x = fmaf(K * K, s3.x, fmaf(-(2 * K + 1), q3.x, 2 * qq3.x));
  const float u4y = fmaf(K * K, s3.y, fmaf(-(2 * K + 1), q3.y, 2 * qq3.y));
  m[0] = s1.x + s1.y;
  m[1] = s2.x + s2.y;
  m[2] = s3.x + s3.y;
  m[3] = s4.x + s4.y;
  m[4] = s5.x + s5.y;
  m[5] = s6.x + s6.y;
  m[6] = u1x + fmaf(K, s2.y, u1y);
  m[7] = u2x + fmaf(K, s3.y, u2y);
  m[8] = u3x + fmaf(K, s5.y, u3y);
  m[9] = u4x + fmaf(K * K, s3.y, fmaf(2 * K, u2y, u4y));
}

// fp32 two-column sweep: a thread owns grid columns col, col+1 and keeps
// them as the two lanes of packed f32x2 registers.  Per frame row it reads
// (F[col], F[col+1]) as one 8-byte load plus F[col+2] (half the shared-memory
// loads of one column per thread); the shifted pairs (P1, P2), (D1, D2) are
// assembled with moves.  m[c] are column c's ten sums (same per-lane
// operation order as sweep()).
#ifndef CT_MOM_SCALAR_H
#define CT_MOM_SCALAR_H 1
#endif
template <int BR, bool CHECK, int BC>
__device__ __forceinline__ void sweep_c2(const float* __restrict__ A, const float* __restrict__ B, int col, int r_beg,
                                         int r_end, float (&m)[2][10]) {
  float2 s1 = {0, 0}, s2 = {0, 0}, s3 = {0, 0}, s4 = {0, 0}, s5 = {0, 0}, s6 = {0, 0};
  float2 q2 = {0, 0}, q3 = {0, 0}, q5 = {0, 0}, qq3 = {0, 0};
  float2 hP, dP, sD;
#if CT_MOM_SCALAR_H
  // The horizontal combinations as scalar adds written straight into the pair
  // registers: a packed add holds the issue port as long as two scalar ones, and
  // the shifted operand pairs (P1, P2), (D1, D2) no longer have to be assembled
  // with moves.
  auto row = [&](int r, float2& nhP, float2& ndP, float2& nsD) {
    const float2 a01 = *reinterpret_cast<const float2*>(A + r * BC + col);
    const float2 b01 = *reinterpret_cast<const float2*>(B + r * BC + col);
    const float a2 = A[r * BC + col + 2], b2 = B[r * BC + col + 2];
    const float2 P01 = f2add(a01, b01);
    const float2 D01 = f2sub(b01, a01);
    const float P2 = a2 + b2, D2 = b2 - a2;
    nhP = make_float2(P01.x + P01.y, P01.y + P2);
    ndP = make_float2(P01.y - P01.x, P2 - P01.y);
    nsD = make_float2(D01.x + D01.y, D01.y + D2);
  };
  row(0, hP, dP, sD);
#pragma unroll
  for (int r = 1; r <= BR; ++r) {
    float2 nhP, ndP, nsD;
    row(r, nhP, ndP, nsD);
#else
  auto row = [&](int r, float2& P01, float2& P12, float2& D01, float2& D12) {
    const float2 a01 = *reinterpret_cast<const float2*>(A + r * BC + col);
    const float2 b01 = *reinterpret_cast<const float2*>(B + r * BC + col);
    const float a2 = A[r * BC + col + 2], b2 = B[r * BC + col + 2];
    P01 = f2add(a01, b01);
    D01 = f2sub(b01, a01);
    P12 = make_float2(P01.y, a2 + b2);
    D12 = make_float2(D01.y, b2 - a2);
  };
  {
    float2 P01, P12, D01, D12;
    row(0, P01, P12, D01, D12);
    hP = f2add(P01, P12);
    dP = f2sub(P12, P01);
    sD = f2add(D01, D12);
  }
#pragma unroll
  for (int r = 1; r <= BR; ++r) {
    float2 P01, P12, D01, D12;
    row(r, P01, P12, D01, D12);
    const float2 nhP = f2add(P01, P12), ndP = f2sub(P12, P01), nsD = f2add(D01, D12);
#endif
    if (!CHECK || (r >= r_beg && r <= r_end)) {
      const float2 ex = f2add(dP, ndP), ey = f2sub(nhP, hP), et = f2add(sD, nsD);
      s1 = f2fma(ex, ex, s1);
      s2 = f2fma(ex, ey, s2);
      s3 = f2fma(ey, ey, s3);
      s4 = f2fma(ex, et, s4);
      s5 = f2fma(ey, et, s5);
      s6 = f2fma(et, et, s6);
    }
    if (r == 1) {
      q2 = s2;
      q3 = s3;
      q5 = s5;
      qq3 = s3;
    } else {
      q2 = f2add(q2, s2);
      q3 = f2add(q3, s3);
      q5 = f2add(q5, s5);
      qq3 = f2add(qq3, q3);
    }
    hP = nhP;
    dP = ndP;
    sD = nsD;
  }
  constexpr float K = float(BR);
  const float2 S[6] = {s1, s2, s3, s4, s5, s6};
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    auto L = [&](float2 v) { return c ? v.y : v.x; };
#pragma unroll
    for (int k = 0; k < 6; ++k) m[c][k] = L(S[k]);
    m[c][6] = fmaf(K, L(s2), -L(q2));
    m[c][7] = fmaf(K, L(s3), -L(q3));
    m[c][8] = fmaf(K, L(s5), -L(q5));
    m[c][9] = fmaf(K * K, L(s3), fmaf(-(2 * K + 1), L(q3), 2 * L(qq3)));
  }
}

// fp32 four-column sweep (CT_MOM_FOUR_COL_F32): a thread owns grid columns
// col..col+3 as two packed f32x2 column pairs; per frame row one 16-byte load
// gives F[col..col+3] and a 4-byte load F[col+4] (a quarter of the loads per
// pixel of one column per thread), the shifted pairs (x+1, x+2), (x+3, x+4)
// are assembled with moves, and the per-pair epilogue and warp reduction are
// paid once per four columns.  Per-lane operation order is sweep()'s.
template <int BR, bool CHECK, int BC>
__device__ __forceinline__ void sweep_c4(const float* __restrict__ A, const float* __restrict__ B, int col, int r_beg,
                                         int r_end, float (&m)[4][10]) {
  float2 s1[2], s2[2], s3[2], s4[2], s5[2], s6[2], q2[2], q3[2], q5[2], qq3[2], hP[2], dP[2], sD[2];
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    s1[p] = s2[p] = s3[p] = s4[p] = s5[p] = s6[p] = make_float2(0.f, 0.f);
    q2[p] = q3[p] = q5[p] = qq3[p] = make_float2(0.f, 0.f);
  }
  auto row = [&](int r, float2 (&nhP)[2], float2 (&ndP)[2], float2 (&nsD)[2]) {
    const float4 a = *reinterpret_cast<const float4*>(A + r * BC + col);
    const float4 b = *reinterpret_cast<const float4*>(B + r * BC + col);
    const float a4 = A[r * BC + col + 4], b4 = B[r * BC + col + 4];
    const float2 P01 = f2add(make_float2(a.x, a.y), make_float2(b.x, b.y));
    const float2 P23 = f2add(make_float2(a.z, a.w), make_float2(b.z, b.w));
    const float2 D01 = f2sub(make_float2(b.x, b.y), make_float2(a.x, a.y));
    const float2 D23 = f2sub(make_float2(b.z, b.w), make_float2(a.z, a.w));
    const float2 P12 = make_float2(P01.y, P23.x), P34 = make_float2(P23.y, a4 + b4);
    const float2 D12 = make_float2(D01.y, D23.x), D34 = make_float2(D23.y, b4 - a4);
    nhP[0] = f2add(P01, P12);
    ndP[0] = f2sub(P12, P01);
    nsD[0] = f2add(D01, D12);
    nhP[1] = f2add(P23, P34);
    ndP[1] = f2sub(P34, P23);
    nsD[1] = f2add(D23, D34);
  };
  row(0, hP, dP, sD);
#pragma unroll
  for (int r = 1; r <= BR; ++r) {
    float2 nhP[2], ndP[2], nsD[2];
    row(r, nhP, ndP, nsD);
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      if (!CHECK || (r >= r_beg && r <= r_end)) {
        const float2 ex = f2add(dP[p], ndP[p]), ey = f2sub(nhP[p], hP[p]), et = f2add(sD[p], nsD[p]);
        s1[p] = f2fma(ex, ex, s1[p]);
        s2[p] = f2fma(ex, ey, s2[p]);
        s3[p] = f2fma(ey, ey, s3[p]);
        s4[p] = f2fma(ex, et, s4[p]);
        s5[p] = f2fma(ey, et, s5[p]);
        s6[p] = f2fma(et, et, s6[p]);
      }
      if (r == 1) {
        q2[p] = s2[p];
        q3[p] = s3[p];
        q5[p] = s5[p];
        qq3[p] = s3[p];
      } else {
        q2[p] = f2add(q2[p], s2[p]);
        q3[p] = f2add(q3[p], s3[p]);
        q5[p] = f2add(q5[p], s5[p]);
        qq3[p] = f2add(qq3[p], q3[p]);
      }
      hP[p] = nhP[p];
      dP[p] = ndP[p];
      sD[p] = nsD[p];
    }
  }
  constexpr float K = float(BR);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int p = c >> 1;
    auto L = [&](float2 v) { return (c & 1) ? v.y : v.x; };
    m[c][0] = L(s1[p]); m[c][1] = L(s2[p]); m[c][2] = L(s3[p]);
    m[c][3] = L(s4[p]); m[c][4] = L(s5[p]); m[c][5] = L(s6[p]);
    m[c][6] = fmaf(K, L(s2[p]), -L(q2[p]));
    m[c][7] = fmaf(K, L(s3[p]), -L(q3[p]));
    m[c][8] = fmaf(K, L(s5[p]), -L(q5[p]));
    m[c][9] = fmaf(K * K, L(s3[p]), fmaf(-(2 * K + 1), L(q3[p]), 2 * L(qq3[p])));
  }
}

// fp64 two-column sweep (CT_MOM_TWO_COL_F64): a thread owns grid columns
// col, col+1; per frame row one 16-byte load gives (F[col], F[col+1]) and an
// 8-byte load F[col+2], and the middle column's time sum/difference is shared
// (19 FP64 operations per grid pixel instead of 20).  Each column keeps
// sweep()'s per-lane operation order and hands back sweep<RAW>'s raw running
// sums, so thread_sums<RAW> folds it exactly like the one-column path.  With
// twice the pixels per lane, the per-pair warp reduction costs half as much
// per pixel.
template <int BR, bool CHECK, int BC>
__device__ __forceinline__ void sweep_c2d(const double* __restrict__ A, const double* __restrict__ B, int col,
                                          int r_beg, int r_end, double (&m)[2][10]) {
  double s1[2] = {0, 0}, s2[2] = {0, 0}, s3[2] = {0, 0}, s4[2] = {0, 0}, s5[2] = {0, 0}, s6[2] = {0, 0};
  double q2[2] = {0, 0}, q3[2] = {0, 0}, q5[2] = {0, 0}, qq3[2] = {0, 0};
  double hP[2], dP[2], sD[2];
  auto row = [&](int r, double (&nhP)[2], double (&ndP)[2], double (&nsD)[2]) {
    const double2 a01 = *reinterpret_cast<const double2*>(A + r * BC + col);
    const double2 b01 = *reinterpret_cast<const double2*>(B + r * BC + col);
    const double a2 = A[r * BC + col + 2], b2 = B[r * BC + col + 2];
    const double P0 = a01.x + b01.x, P1 = a01.y + b01.y, P2 = a2 + b2;
    const double D0 = b01.x - a01.x, D1 = b01.y - a01.y, D2 = b2 - a2;
    nhP[0] = P0 + P1;
    ndP[0] = P1 - P0;
    nsD[0] = D0 + D1;
    nhP[1] = P1 + P2;
    ndP[1] = P2 - P1;
    nsD[1] = D1 + D2;
  };
  row(0, hP, dP, sD);
#pragma unroll
  for (int r = 1; r <= BR; ++r) {
    double nhP[2], ndP[2], nsD[2];
    row(r, nhP, ndP, nsD);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      if (!CHECK || (r >= r_beg && r <= r_end)) {
        const double ex = dP[c] + ndP[c];
        const double ey = nhP[c] - hP[c];
        const double et = sD[c] + nsD[c];
        s1[c] = fma(ex, ex, s1[c]);
        s2[c] = fma(ex, ey, s2[c]);
        s3[c] = fma(ey, ey, s3[c]);
        s4[c] = fma(ex, et, s4[c]);
        s5[c] = fma(ey, et, s5[c]);
        s6[c] = fma(et, et, s6[c]);
      }
      if (r == 1) {
        q2[c] = s2[c];
        q3[c] = s3[c];
        q5[c] = s5[c];
        qq3[c] = s3[c];
      } else {
        q2[c] += s2[c];
        q3[c] += s3[c];
        q5[c] += s5[c];
        qq3[c] += q3[c];
      }
      hP[c] = nhP[c];
      dP[c] = ndP[c];
      sD[c] = nsD[c];
    }
  }
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    m[c][0] = s1[c]; m[c][1] = s2[c]; m[c][2] = s3[c]; m[c][3] = s4[c]; m[c][4] = s5[c]; m[c][5] = s6[c];
    m[c][6] = q2[c]; m[c][7] = q3[c]; m[c][8] = q5[c]; m[c][9] = qq3[c];
  }
}

// This thread's ten normal-system sums for one pair (order m00 m01 m02 m11
// m12 m22 r0 r1 r2 et2, rhs not yet negated) from its per-column sweep
// sums: the band-relative y weights are shifted by the absolute centred y
// of the thread's first row (yc0) and G = xc Ex + yc Ey is expanded with
// the column's xc.
// RAW: m[6..9] are the running sums (Q2, Q3, Q5, QQ3) of a K-row sweep; with
// Y = yc0 + K, U1 = Y S2 - Q2, U2 = Y S3 - Q3, U3 = Y S5 - Q5 and
// U4 = Y^2 S3 - (2Y + 1) Q3 + 2 QQ3 (sweep()'s identities with the shift folded in).
// ALLIN: every column of every lane of the warp is inside the window (all
// warps but a tile's first and last): no zero-initialised outputs, no
// divergent region around the fold.
template <typename ACC, int CPT, typename E, bool RAW = false, int K = 0, bool ALLIN = false>
__device__ __forceinline__ void thread_sums(const ACC (&mc)[CPT][10], const bool (&in_col)[CPT],
                                            const double (&xc)[CPT], double yc0d, E (&o)[10]) {
  const E yc0 = (E)yc0d;  // centred coordinates are half-integers: exact in f32 and f64
  const E Y = yc0 + E(K);
  if constexpr (!ALLIN || CPT > 1) {
#pragma unroll
    for (int q = 0; q < 10; ++q) o[q] = E(0);
  }
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    if (ALLIN || in_col[c]) {
      const ACC(&m)[10] = mc[c];
      const E S1 = m[0], S2 = m[1], S3 = m[2], S4 = m[3], S5 = m[4], S6 = m[5];
      E U1, U2, U3, U4;
      if constexpr (RAW) {
        U1 = fma(Y, S2, -(E)m[6]);
        U2 = fma(Y, S3, -(E)m[7]);
        U3 = fma(Y, S5, -(E)m[8]);
        U4 = fma(Y * Y, S3, fma(-(E(2) * Y + E(1)), (E)m[7], (E)m[9] + (E)m[9]));
      } else {
        U1 = fma(yc0, S2, (E)m[6]);
        U2 = fma(yc0, S3, (E)m[7]);
        U3 = fma(yc0, S5, (E)m[8]);
        U4 = fma(yc0 * yc0, S3, fma(E(2) * yc0, (E)m[7], (E)m[9]));
      }
      const E X = (E)xc[c];
      const E v[10] = {S1, S2, fma(X, S1, U1), S3, fma(X, S2, U2), fma(X * X, S1, fma(E(2) * X, U1, U4)),
                       S4, S5, fma(X, S4, U3), S6};
#pragma unroll
      for (int q = 0; q < 10; ++q) o[q] = CPT == 1 ? v[q] : o[q] + v[q];
    }
  }
}

// Sum each of ten values over the 32 lanes of a warp with a fixed
// transpose-reduce butterfly (10 -> 5 -> 3 -> 2 -> 1 values per lane over
// xor 16, 8, 4, 2, 1; 12 shuffles and 12 adds per lane instead of 50).  On
// return lane l holds the warp total of value `idx` (idx = -1: padding);
// both lanes of an even/odd pair hold the same value.  The order of the adds
// depends only on the lane, so the result is bit-reproducible.
template <typename E>
__device__ __forceinline__ E warp_reduce10(const E (&o)[10], int lane, int& idx) {
  constexpr unsigned kFull = 0xffffffffu;
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
  E r1[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const E keep = b4 ? o[k + 5] : o[k], send = b4 ? o[k] : o[k + 5];
    r1[k] = keep + __shfl_xor_sync(kFull, send, 16);
  }
  E r2[3];  // b3 = 0 keeps r1[0..2], b3 = 1 keeps r1[3..4] (+ padding)
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const E lo = r1[k], hi = k < 2 ? r1[3 + k] : E(0);
    r2[k] = (b3 ? hi : lo) + __shfl_xor_sync(kFull, b3 ? lo : hi, 8);
  }
  E r3[2];  // b2 = 0 keeps r2[0..1], b2 = 1 keeps r2[2] (+ padding)
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const E lo = r2[k], hi = k < 1 ? r2[2] : E(0);
    r3[k] = (b2 ? hi : lo) + __shfl_xor_sync(kFull, b2 ? lo : hi, 4);
  }
  const E r4 = (b1 ? r3[1] : r3[0]) + __shfl_xor_sync(kFull, b1 ? r3[0] : r3[1], 2);
  const E r5 = r4 + __shfl_xor_sync(kFull, r4, 1);
  // which value this lane ended with: list start/length after each split
  int st = b4 ? 5 : 0, len = 5;
  st += b3 ? 3 : 0;
  len = b3 ? 2 : 3;
  st += b2 ? 2 : 0;
  len = b2 ? len - 2 : min(len, 2);
  idx = (b1 ? len >= 2 : len >= 1) ? st + (b1 ? 1 : 0) : -1;
  return r5;
}

// CT_MOM_EARLY_REL: a warp releases frame i right after its sweep (the
// atomic's result is consumed after the per-thread epilogue, so its latency is
// covered and the refill is issued before the warp reduction instead of after
// it); the combine then lags one more pair (a released frame no longer implies
// that pair's deposit, only the previous pair's).
#ifndef CT_MOM_EARLY_REL
#define CT_MOM_EARLY_REL 0  // measured: no change on cfg2 (1.815 vs 1.812 ms) or 1080p fp32 (0.960 vs 0.955 ms); kept as an option
#endif
template <typename T, int BR, int NB, int BC, int NT>
struct SmemWS {  // warp-streaming kernel: NB frame-band buffers + per-buffer release counters + warp partials
  static constexpr int NW = NT / 32;
  // pair slots for the warp partials: 2 NB pairs can be live (see the kernel)
  static constexpr int NS = CT_MOM_EARLY_REL ? 2 * NB : (2 * NB - 2 > 3 ? 2 * NB - 2 : 3);
  static constexpr size_t buf_elems = (size_t)(BR + 1) * BC + 8;
  static constexpr size_t buf_bytes = (buf_elems * sizeof(T) + 127) & ~size_t(127);
  static constexpr size_t bars_off = NB * buf_bytes;
  static constexpr size_t rel_off = bars_off + 8 * NB;
  static constexpr size_t part_off = (rel_off + 4 * NB + 15) & ~size_t(15);
  static constexpr size_t total = part_off + (size_t)NS * NW * 10 * sizeof(double);
};

// Warp-streaming variant of the fused moments kernel (used whenever the
// frames admit a TMA map): no CTA-wide barrier in the steady state.
//   * Each warp waits on the TMA mbarriers of the two frames of a pair by
//     itself; when it has finished with frame i it bumps that buffer's
//     release counter, and the last of the NW warps to release it issues the
//     TMA of frame i + NB into the freed buffer.
//   * A warp's 32 lanes reduce their ten sums with warp_reduce10 and deposit
//     one 10-value partial per warp in pair slot i % NS.  Pair i - (NB - 1)
//     is complete once a warp holds frame i + 1 (that load waited for every
//     warp's release of frame i + 1 - NB, which follows its deposit), so warp
//     (i - (NB - 1)) % NW adds its NW partials in a fixed pairwise tree and
//     writes the band's partial; the last NB - 1 pairs are combined after a
//     barrier at the end.  The add order is fixed: results are
//     bit-reproducible.  No arrival counter is needed and the combine rotates
//     over the warps instead of delaying the slowest one (each per-pair delay
//     of one warp holds up every warp's next refill: counter-based combining
//     by the last arriver was 1.3 % slower on cfg2).
//   * Pairs i - (NB - 1) .. i + NB - 2 can hold live partials, so NS = 2 NB - 2.
//   * RS row splits: the 32 / RS lanes of a warp's row group own consecutive
//     column groups (CPT columns each) and the RS groups split the band rows,
//     so fp32 bands run 256 threads (16 warps per SM) with two columns per
//     thread.
#ifndef CT_MOM_MINB64
#define CT_MOM_MINB64 0
#endif
#ifndef CT_MOM_MINB32
#define CT_MOM_MINB32 3
#endif
// resident CTAs per SM the register budget is sized for (fp32: CT_MOM_MINB32, see band_rows)
template <typename T, int BC, int RS>
constexpr int ws_min_blocks() {
  return (sizeof(T) == 4 && CT_MOM_MINB32 > 0)   ? CT_MOM_MINB32
         : (sizeof(T) == 8 && CT_MOM_MINB64 > 0) ? CT_MOM_MINB64
                                                 : ((512 / BC) / RS > 0 ? (512 / BC) / RS : 1);
}

template <typename T, int BR, int NB, int BC, int CPT, int RS>
__device__ __forceinline__ void moments_ws_body(const MomentArgs& a, const CUtensorMap* tmap, unsigned char* smem,
                                                int unit, int chunk_idx, int64_t v) {
  using ACC = typename AccT<T>::type;
  constexpr int kThreads = BC / CPT * RS;
  using S = SmemWS<T, BR, NB, BC, kThreads>;
  constexpr int NW = S::NW;
  constexpr int HR = BR / RS;        // band rows per row group
  constexpr int LG = 32 / RS;        // lanes per row group
  static_assert(BR % RS == 0 && 32 % RS == 0, "row split");
  // fp64 sweeps hand back raw running sums (folded in thread_sums)
  constexpr bool kRaw = sizeof(T) == 8;
  auto buf = [&](int k) { return reinterpret_cast<T*>(smem + (size_t)k * S::buf_bytes); };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::bars_off);
  int* rel = reinterpret_cast<int*>(smem + S::rel_off);
  double* part = reinterpret_cast<double*>(smem + S::part_off);

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int band = unit / a.n_ctiles, ctile = unit - band * a.n_ctiles;
  const int gy0 = band * BR;
  const int cx0 = ctile * a.tile_cols;
  const int n_pairs = a.n_frames - 1;
  const int p0 = chunk_idx * a.chunk;
  const int p1 = min(p0 + a.chunk, n_pairs);
  if (p0 >= p1) return;
  const int nload = p1 - p0 + 1;
  constexpr uint32_t kBoxBytes = (uint32_t)((BR + 1) * BC * sizeof(T));

  const int rg = lane / LG;                              // row group of this lane
  const int col = (wid * LG + lane % LG) * CPT;           // first tile column of this thread
  const int r0 = rg * HR;                                 // rows r0+1 .. r0+HR of the band (start row r0)
  bool in_col[CPT];
  double xc[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int gx = cx0 + col + c;
    in_col[c] = col + c < a.tile_cols && gx >= a.border && gx < a.gw - a.border;
    xc[c] = (double)gx - (double)(a.gw - 1) / 2.0;
  }
  const double yc0 = (double)(gy0 + r0) - (double)(a.gh - 1) / 2.0;  // centred y of this thread's first grid row
  bool all_in_t = true;
#pragma unroll
  for (int c = 0; c < CPT; ++c) all_in_t = all_in_t && in_col[c];
  const bool all_in = __all_sync(0xffffffffu, all_in_t);  // warp-uniform: the fold without the column mask
  const int64_t row0 = (v * a.n_frames) * (int64_t)a.h + gy0;
  // thread-local row range [r_beg, r_end] (1..HR) whose grid rows are interior
  const int r_end = min(HR, a.gh - a.border - gy0 - r0);
  const int r_beg = max(1, a.border - gy0 - r0 + 1);

  auto issue = [&](int f) {
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&bars[f % NB], kBoxBytes);
    tma_load_2d(buf(f % NB), tmap, &bars[f % NB], cx0, (int)(row0 + (int64_t)(p0 + f) * a.h));
  };
  if (tid == 0) {
    for (int i = 0; i < NB; ++i) {
      mbar_init(&bars[i], 1);
      rel[i] = 0;
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int f = 0; f < min(NB, nload); ++f) issue(f);

  // band partial of pair p0 + j: the NW warp partials in a fixed pairwise tree
  auto combine = [&](int j) {
    const double* pj = part + (size_t)(j % S::NS) * NW * 10;
    if (lane < 10) {
      double t[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) t[w] = pj[w * 10 + lane];
#pragma unroll
      for (int h = 1; h < NW; h *= 2)
#pragma unroll
        for (int w = 0; w + h < NW; w += 2 * h) t[w] += t[w + h];
      const double acc = t[0] * 0.0625;  // undo the 4x stencil scaling of both factors
      a.partials[((v * n_pairs + p0 + j) * a.units + unit) * 10 + lane] = (lane >= 6 && lane <= 8) ? -acc : acc;
    }
  };
  for (int i = 0; i < p1 - p0; ++i) {
    const int p = p0 + i;
    if (i == 0) mbar_wait(&bars[0], 0u);  // later pairs: frame i arrived as frame B of pair i - 1
    mbar_wait(&bars[(i + 1) % NB], (uint32_t)(((i + 1) / NB) & 1));
    const T* A = buf(i % NB);
    const T* B = buf((i + 1) % NB);
    if (a.dec) {
      write_dec<T, BR, kThreads, BC>(a, A, v, p, gy0, cx0, tid);
      if (p1 == n_pairs && i == p1 - p0 - 1) write_dec<T, BR, kThreads, BC>(a, B, v, p1, gy0, cx0, tid);
    }
    const T* Ar = A + r0 * BC;
    const T* Br = B + r0 * BC;
    ACC mc[CPT][10];
    if constexpr (CPT == 2 && sizeof(T) == 8) {
      if (r_beg <= 1 && r_end >= HR)
        sweep_c2d<HR, false, BC>(reinterpret_cast<const double*>(Ar), reinterpret_cast<const double*>(Br), col, 1,
                                 HR, mc);
      else
        sweep_c2d<HR, true, BC>(reinterpret_cast<const double*>(Ar), reinterpret_cast<const double*>(Br), col, r_beg,
                                r_end, mc);
    } else if constexpr (CPT == 4) {
      if (r_beg <= 1 && r_end >= HR)
        sweep_c4<HR, false, BC>(reinterpret_cast<const float*>(Ar), reinterpret_cast<const float*>(Br), col, 1, HR,
                                mc);
      else
        sweep_c4<HR, true, BC>(reinterpret_cast<const float*>(Ar), reinterpret_cast<const float*>(Br), col, r_beg,
                               r_end, mc);
    } else if constexpr (CPT == 2) {
      if (r_beg <= 1 && r_end >= HR)
        sweep_c2<HR, false, BC>(reinterpret_cast<const float*>(Ar), reinterpret_cast<const float*>(Br), col, 1, HR,
                                mc);
      else
        sweep_c2<HR, true, BC>(reinterpret_cast<const float*>(Ar), reinterpret_cast<const float*>(Br), col, r_beg,
                               r_end, mc);
    } else {
      ACC(&m)[10] = mc[0];
      if (r_beg <= 1 && r_end >= HR) {
        if constexpr (sizeof(T) == 4 && kPackedF32 && HR % 2 == 0)
          sweep_x2<HR, BC>(reinterpret_cast<const float*>(Ar), reinterpret_cast<const float*>(Br), col, m);
        else
          sweep<T, HR, false, BC, kRaw>(Ar, Br, col, 1, HR, m);
      } else {
        sweep<T, HR, true, BC, kRaw>(Ar, Br, col, r_beg, r_end, m);
      }
    }
    // fp32 frames: per-thread epilogue and warp reduction in fp32 (the FP64
    // pipe is half rate); fp64 frames: fp64 throughout
    using E = typename std::conditional<sizeof(T) == 4, float, double>::type;
#ifdef CT_PROBE_NO_EPI  // probing only: the per-pair epilogue and warp reduction removed (wrong sums)
    {
      ACC acc = 0;
#pragma unroll
      for (int c = 0; c < CPT; ++c)
#pragma unroll
        for (int q = 0; q < 10; ++q) acc += mc[c][q];
      double* ps = part + (size_t)(i % S::NS) * NW * 10;
      if (lane < 10) ps[wid * 10 + lane] = (double)acc;
    }
#else
    E o[10];
#if CT_MOM_EARLY_REL
    // frame p0 + i (buffer i % NB) is dead for this warp once the sweep's
    // loads have returned (the sums above depend on all of them)
    int relv = 0;
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      relv = atomicAdd(&rel[i % NB], 1);
    }
#endif
    if (all_in)
      thread_sums<ACC, CPT, E, kRaw, HR, true>(mc, in_col, xc, yc0, o);
    else
      thread_sums<ACC, CPT, E, kRaw, HR>(mc, in_col, xc, yc0, o);
#if CT_MOM_EARLY_REL
    // the last warp to release the buffer refills it with frame p0 + i + NB
    if (lane == 0 && (relv % NW) == NW - 1 && i + NB < nload) issue(i + NB);
    __syncwarp();
#endif
    int idx;
    const double wsum = (double)warp_reduce10<E>(o, lane, idx);
    double* ps = part + (size_t)(i % S::NS) * NW * 10;
    if ((lane & 1) == 0 && idx >= 0) ps[wid * 10 + idx] = wsum;
#endif
#if CT_MOM_EARLY_REL && !defined(CT_PROBE_NO_EPI)
    // Pair i - NB is complete: frame i + 1 (awaited above) was loaded only
    // after every warp released frame i + 1 - NB, i.e. finished the sweep of
    // pair i + 1 - NB, which follows its deposit of pair i - NB.  The combine
    // rotates over the warps: no arrival counter, no extra work on one warp.
    if (i >= NB && wid == (i - NB) % NW) {
      __threadfence_block();
      combine(i - NB);
    }
  }
  // the last NB pairs
  __syncthreads();
  for (int j = max(0, p1 - p0 - NB) + wid; j < p1 - p0; j += NW) combine(j);
}
#else
    // Pair i - (NB - 1) is complete: frame i + 1 (awaited above) was loaded
    // only after every warp released frame i + 1 - NB, which each warp does
    // after depositing that pair.  Its combine rotates over the warps, so no
    // arrival counter is needed and the slowest warp carries no extra work.
    if (i >= NB - 1 && wid == (i - (NB - 1)) % NW) {
      __threadfence_block();
      combine(i - (NB - 1));
    }
    __syncwarp();
    // frame p0 + i (buffer i % NB) is dead for this warp: the last warp to
    // release it refills the buffer with frame p0 + i + NB
    if (lane == 0) {
      __threadfence_block();
      if ((atomicAdd(&rel[i % NB], 1) % NW) == NW - 1 && i + NB < nload) issue(i + NB);
    }
  }
  // the last NB - 1 pairs
  __syncthreads();
  for (int j = max(0, p1 - p0 - (NB - 1)) + wid; j < p1 - p0; j += NW) combine(j);
}
#endif

template <typename T, int BR, int NB, int BC, int CPT, int RS>
__global__ void __launch_bounds__(BC / CPT * RS, ws_min_blocks<T, BC, RS>())
    ttc_moments_ws_kernel(const MomentArgs a, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) unsigned char smem[];
  moments_ws_body<T, BR, NB, BC, CPT, RS>(a, &tmap, smem, blockIdx.x, blockIdx.y, blockIdx.z);
}

// Several pyramid levels in one launch (the small levels alone cannot fill
// the GPU): a 1-D grid whose CTAs are the concatenated (unit, chunk, video)
// grids of the levels, largest level first.
constexpr int kMaxLevels = kMomentLevelsPerLaunch;
struct LevelsArgs {
  CUtensorMap tmap[kMaxLevels];
  MomentArgs a[kMaxLevels];
  int64_t cta_end[kMaxLevels];
  int n;
};

template <typename T, int BR, int NB, int BC, int CPT, int RS>
__global__ void __launch_bounds__(BC / CPT * RS, ws_min_blocks<T, BC, RS>())
    ttc_moments_levels_kernel(const __grid_constant__ LevelsArgs m) {
  extern __shared__ __align__(128) unsigned char smem[];
  int l = 0;
  while (l + 1 < m.n && (int64_t)blockIdx.x >= m.cta_end[l]) ++l;
  const int64_t local = (int64_t)blockIdx.x - (l ? m.cta_end[l - 1] : 0);
  const MomentArgs& a = m.a[l];
  const int unit = (int)(local % a.units);
  const int64_t rest = local / a.units;
  const int n_chunks = (a.n_frames - 1 + a.chunk - 1) / a.chunk;
  moments_ws_body<T, BR, NB, BC, CPT, RS>(a, &m.tmap[l], smem, unit, (int)(rest % n_chunks), rest / n_chunks);
}

template <typename T, int BR, int NB, int BC, int CPT>
__global__ void __launch_bounds__(BC / CPT, 512 / BC) ttc_moments_kernel(const MomentArgs a,
                                                                        const __grid_constant__ CUtensorMap tmap) {
  using ACC = typename AccT<T>::type;
  constexpr int kThreads = BC / CPT;
  using S = Smem<T, BR, NB, BC, kThreads>;
  static_assert(CPT == 1 || sizeof(T) == 4, "two columns per thread is the fp32 path");
  constexpr int kRedSeg = S::seg;
  extern __shared__ __align__(128) unsigned char smem[];
  auto buf = [&](int k) { return reinterpret_cast<T*>(smem + (size_t)k * S::buf_bytes); };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::bars_off);
  double* part = reinterpret_cast<double*>(smem + S::part_off);

  const int tid = threadIdx.x;
  const int unit = blockIdx.x;
  const int band = unit / a.n_ctiles, ctile = unit - band * a.n_ctiles;
  const int gy0 = band * BR;              // first grid row == first frame row of the band
  const int cx0 = ctile * a.tile_cols;     // first grid column == first frame column
  const int64_t v = blockIdx.z;
  const int n_pairs = a.n_frames - 1;
  const int p0 = blockIdx.y * a.chunk;
  const int p1 = min(p0 + a.chunk, n_pairs);  // pairs [p0, p1) -> frames p0..p1
  if (p0 >= p1) return;
  const int nload = p1 - p0 + 1;
  constexpr uint32_t kBoxBytes = (uint32_t)((BR + 1) * BC * sizeof(T));

  const int col = tid * CPT;  // first tile column of this thread
  bool in_col[CPT];
  double xc[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int gx = cx0 + col + c;
    in_col[c] = col + c < a.tile_cols && gx >= a.border && gx < a.gw - a.border;
    xc[c] = (double)gx - (double)(a.gw - 1) / 2.0;
  }
  const double yc0 = (double)gy0 - (double)(a.gh - 1) / 2.0;    // centred y of grid row gy0
  const int64_t row0 = (v * a.n_frames) * (int64_t)a.h + gy0;  // band row of frame p: row0 + p*h
  // band-local frame-row range r in [r_beg, r_end] whose grid row gy0 + r - 1 is interior
  const int r_end = min(BR, a.gh - a.border - gy0);
  const int r_beg = max(1, a.border - gy0 + 1);

  auto issue = [&](int f) {  // frame p0+f -> buffer f%3
    T* dst = buf(f % NB);
    const int64_t grow = row0 + (int64_t)(p0 + f) * a.h;
    if (a.use_tma) {
      if (tid == 0) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bars[f % NB], kBoxBytes);
        tma_load_2d(dst, &tmap, &bars[f % NB], cx0, (int)grow);
      }
    } else {
      const T* src = reinterpret_cast<const T*>(a.frames) + grow * a.w;
      const int64_t rows_left = a.n_videos * a.n_frames * (int64_t)a.h - grow;
      for (int idx = tid; idx < (BR + 1) * BC; idx += kThreads) {
        const int r = idx / BC, c = idx - r * BC;
        T val = T(0);
        if (r < rows_left && cx0 + c < a.w) val = src[(int64_t)r * a.w + cx0 + c];
        dst[idx] = val;
      }
    }
  };

  if (a.use_tma) {
    if (tid == 0) {
      for (int i = 0; i < NB; ++i) mbar_init(&bars[i], 1);
      mbar_fence_init();
    }
    __syncthreads();
    for (int f = 0; f < min(NB, nload); ++f) issue(f);
  } else {
    issue(0);
    issue(1);
    __syncthreads();
  }

  for (int i = 0; i < p1 - p0; ++i) {
    const int p = p0 + i;
    if (a.use_tma) {
      mbar_wait(&bars[i % NB], (uint32_t)((i / NB) & 1));
      mbar_wait(&bars[(i + 1) % NB], (uint32_t)(((i + 1) / NB) & 1));
    }
    const T* A = buf(i % NB);
    const T* B = buf((i + 1) % NB);

    if (a.dec) {  // frames p0..p1-1 belong to this chunk (the last chunk also owns frame p1)
      write_dec<T, BR, kThreads, BC>(a, A, v, p, gy0, cx0, tid);
      if (p1 == n_pairs && i == p1 - p0 - 1) write_dec<T, BR, kThreads, BC>(a, B, v, p1, gy0, cx0, tid);
    }
    ACC mc[CPT][10];
    if constexpr (CPT == 2) {
      if (r_beg <= 1 && r_end >= BR)
        sweep_c2<BR, false, BC>(reinterpret_cast<const float*>(A), reinterpret_cast<const float*>(B), col, 1, BR, mc);
      else
        sweep_c2<BR, true, BC>(reinterpret_cast<const float*>(A), reinterpret_cast<const float*>(B), col, r_beg, r_end,
                               mc);
    } else {
      ACC(&m)[10] = mc[0];
      if (r_beg <= 1 && r_end >= BR) {
        if constexpr (sizeof(T) == 4 && kPackedF32)
          sweep_x2<BR, BC>(A, B, col, m);
        else
          sweep<T, BR, false, BC>(A, B, col, 1, BR, m);
      } else {
        sweep<T, BR, true, BC>(A, B, col, r_beg, r_end, m);
      }
    }

    // this thread's ten sums, order m00 m01 m02 m11 m12 m22 r0 r1 r2 et2 (rhs not yet negated)
    double o[10];
#pragma unroll
    for (int q = 0; q < 10; ++q) o[q] = 0.0;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if (in_col[c]) {
        const ACC(&m)[10] = mc[c];
        const double S1 = m[0], S2 = m[1], S3 = m[2], S4 = m[3], S5 = m[4], S6 = m[5];
        const double U1 = fma(yc0, S2, (double)m[6]);
        const double U2 = fma(yc0, S3, (double)m[7]);
        const double U3 = fma(yc0, S5, (double)m[8]);
        const double U4 = fma(yc0 * yc0, S3, fma(2.0 * yc0, (double)m[7], (double)m[9]));
        const double X = xc[c];
        const double v[10] = {S1, S2, fma(X, S1, U1), S3, fma(X, S2, U2), fma(X * X, S1, fma(2.0 * X, U1, U4)),
                              S4, S5, fma(X, S4, U3), S6};
#pragma unroll
        for (int q = 0; q < 10; ++q) o[q] = CPT == 1 ? v[q] : o[q] + v[q];
      }
    }
    double* red = reinterpret_cast<double*>(const_cast<T*>(A));  // frame p0+i is dead after the sweep
    if (S::half_red) {
#pragma unroll
      for (int q = 0; q < 10; ++q) o[q] += __shfl_xor_sync(0xffffffffu, o[q], 1);
    }
    __syncthreads();  // every thread is done reading A and B for this pair
    if (!S::half_red || (tid & 1) == 0) {
      const int slot = S::half_red ? tid >> 1 : tid;
#pragma unroll
      for (int q = 0; q < 10; ++q) red[q * S::red_n + slot] = o[q];
    }
    __syncthreads();
    if (tid < 10 * kRedSeg) {  // stage 1: value q, segment g sums slots g, g+16, g+32, ...
      const int q = tid / kRedSeg, g = tid % kRedSeg;
      const double* rq = red + q * S::red_n + g;
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < S::red_n / kRedSeg; ++j) acc += rq[j * kRedSeg];
      part[q * kRedSeg + g] = acc;
    }
    __syncthreads();  // scratch consumed: buffer i%NB may be refilled
    if (a.use_tma) {
      if (i + NB < nload) issue(i + NB);
    } else if (i + 2 < nload) {
      issue(i + 2);  // buffer (i+2)%NB last held frame p0+i+2-NB <= p0+i-1
    }
    if (tid < 10) {
      double acc = 0.0;
#pragma unroll
      for (int g = 0; g < kRedSeg; ++g) acc += part[tid * kRedSeg + g];
      acc *= 0.0625;  // undo the 4x stencil scaling of both factors
      // rhs entries are the negated sums (ttc.py:119)
      a.partials[((v * n_pairs + p) * a.units + unit) * 10 + tid] = (tid >= 6 && tid <= 8) ? -acc : acc;
    }
    if (!a.use_tma) __syncthreads();
  }
}

// sums[sys] = fixed-order sum of the `units` band partials of each system.
// One warp per system: lane l adds the partial rows u = l, l+32, ... (each
// row is 10 contiguous doubles, so a warp step reads 32 consecutive rows,
// coalesced), then a fixed butterfly combines the lanes; the order depends
// only on `units`, so results are bit-reproducible.  Persistent: a few
// resident blocks per SM walk the systems.
constexpr int kFinWarps = 8;
__global__ void __launch_bounds__(kFinWarps * 32) moments_finalize_kernel(const double* partials, int64_t n_sys,
                                                                         int units, double count, double* sums) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * kFinWarps;
  for (int64_t sys = (int64_t)blockIdx.x * kFinWarps + (threadIdx.x >> 5); sys < n_sys; sys += nwarps) {
    double acc[10];
#pragma unroll
    for (int q = 0; q < 10; ++q) acc[q] = 0.0;
    for (int u = lane; u < units; u += 32) {
      const double2* r = reinterpret_cast<const double2*>(partials + (sys * units + u) * 10);
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
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < 10; ++q) sums[sys * 11 + q] = acc[q];
      sums[sys * 11 + 10] = count;
    }
  }
}

inline unsigned finalize_grid(int64_t n_sys) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n_sys, kFinWarps), (int64_t)num_sms() * 8));
}

// Band height: 16 rows for f64 (3 x 35 KB buffers, 2 CTAs/SM, FP64-bound);
// 20 rows for f32 (3 x 21 KB, 3 CTAs/SM of 4 warps with <= 170 registers):
// the fp32 kernel is latency-bound; on the full cfg5 stream 20-row bands at
// 12 warps/SM match 22 rows and beat 16-row bands at 4 CTAs/SM (which win on
// a single 128-frame video), 32-row bands at 8 warps/SM and 4-deep rings
// (profiles/r01_moments_probe.md).
#ifndef CT_MOM_BR32
#define CT_MOM_BR32 20
#endif
#ifndef CT_MOM_NB32
#define CT_MOM_NB32 3
#endif
#ifndef CT_MOM_BR64
#define CT_MOM_BR64 16
#endif
#ifndef CT_MOM_NB64
#define CT_MOM_NB64 3
#endif
template <typename T>
constexpr int band_rows() {
  return sizeof(T) == 8 ? CT_MOM_BR64 : CT_MOM_BR32;
}
template <typename T>
constexpr int ring_buffers() {
  return sizeof(T) == 8 ? CT_MOM_NB64 : CT_MOM_NB32;
}

#ifndef CT_MOM_WAVES
#define CT_MOM_WAVES 8
#endif
#ifndef CT_MOM_MIN_CHUNK
#define CT_MOM_MIN_CHUNK 4
#endif
constexpr int kMinChunk = CT_MOM_MIN_CHUNK;  // fewest pairs per CTA chunk (each chunk re-reads one frame)

struct Plan {
  int n_bands, n_ctiles, units, chunk, n_chunks, tile_cols;
};

// Tile width: 256 columns.  128-column tiles (4 CTAs of 4 warps per SM) were
// 4.5 % faster on 1080x1920 fp32 with one column per thread, but with two
// columns per thread (fp32) and for fp64 the 256-column tiles win on wide
// frames too (profiles/r01_moments_probe.md); 128 stays selectable for probing.
inline int pick_bc(int w) {
  (void)w;
  if (const char* e = getenv("CT_MOM_BC")) return atoi(e) == 128 ? 128 : 256;  // probing / tests only
  return 256;
}

template <typename T, int BC>
Plan make_plan(int64_t n_videos, int n_frames, int h, int w) {
  Plan p{};
  constexpr int BR = band_rows<T>();
  const int gh = h - 1, gw = w - 1;
  p.n_bands = (gh + BR - 1) / BR;
  p.tile_cols = gw <= BC - 1 ? BC - 1 : BC - 4;
  p.n_ctiles = (gw + p.tile_cols - 1) / p.tile_cols;
  p.units = p.n_bands * p.n_ctiles;
  const int n_pairs = n_frames - 1;
  // ~4 waves of resident CTAs (2 per SM), but >= kMinChunk pairs per CTA so the
  // one-frame time halo of each chunk stays small
  const int64_t target = (int64_t)num_sms() * CT_MOM_WAVES * ws_min_blocks<T, BC, 1>();  // resident CTAs x waves
  const int64_t per_chunk = std::max<int64_t>(1, (int64_t)p.units * n_videos);
  int64_t chunks = std::max<int64_t>(1, (target + per_chunk - 1) / per_chunk);
  chunks = std::min<int64_t>(chunks, std::max(1, n_pairs / kMinChunk));
  chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, n_pairs));
  p.chunk = (int)((n_pairs + chunks - 1) / chunks);
  p.n_chunks = (n_pairs + p.chunk - 1) / p.chunk;
  return p;
}

template <typename T>
Plan make_plan(int64_t n_videos, int n_frames, int h, int w) {
  return pick_bc(w) == 128 ? make_plan<T, 128>(n_videos, n_frames, h, w) : make_plan<T, 256>(n_videos, n_frames, h, w);
}

template <typename T>
size_t ws_bytes(int64_t n_videos, int n_frames, int h, int w) {
  if (n_frames < 2 || h < 2 || w < 2) return 0;
  const Plan p = make_plan<T>(n_videos, n_frames, h, w);
  return (size_t)n_videos * (n_frames - 1) * p.units * 10 * sizeof(double);
}

#ifndef CT_MOM_TWO_COL_F64
#define CT_MOM_TWO_COL_F64 0
#endif
#ifndef CT_MOM_FOUR_COL_F32
#define CT_MOM_FOUR_COL_F32 0
#endif
// row groups per warp (RS): probing knob for the fp64 two-column sweep (CT_MOM_RS64=2 keeps 256 threads)
#ifndef CT_MOM_RS64
#define CT_MOM_RS64 1
#endif
template <typename T>
constexpr int row_split() {
  return sizeof(T) == 8 ? CT_MOM_RS64 : 1;
}
template <typename T, int BC>
constexpr int cols_per_thread() {
  return (sizeof(T) == 4 && CT_MOM_FOUR_COL_F32 && BC == 256) ? 4
         : (sizeof(T) == 4 && kTwoColF32 && BC == 256)           ? 2
         : (sizeof(T) == 8 && CT_MOM_TWO_COL_F64 && BC == 256)   ? 2
                                                                 : 1;
}
// the CTA-barrier kernel (plain-load fallback) runs fp64 one column per thread
template <typename T, int BC>
constexpr int cols_per_thread_sync() {
  return sizeof(T) == 8 ? 1 : (cols_per_thread<T, BC>() > 2 ? 2 : cols_per_thread<T, BC>());
}

// Kernel arguments and TMA map of one level; returns whether the frames admit
// a TMA map (16-byte aligned base and row pitch), else the LDG-loader kernel runs.
template <typename T, int BC>
bool prep_level(MomentArgs& a, CUtensorMap& tmap, const T* frames, int64_t n_videos, int n_frames, int h, int w,
                int border, double* partials, void* dec, int chunk = 0) {
  constexpr int BR = band_rows<T>();
  const Plan p = make_plan<T, BC>(n_videos, n_frames, h, w);
  a = MomentArgs{};
  a.frames = frames;
  a.partials = partials;
  a.n_videos = n_videos;
  a.n_frames = n_frames;
  a.h = h;
  a.w = w;
  a.gh = h - 1;
  a.gw = w - 1;
  a.border = border;
  a.n_ctiles = p.n_ctiles;
  a.units = p.units;
  a.chunk = chunk > 0 ? std::min(chunk, n_frames - 1) : p.chunk;
  a.tile_cols = p.tile_cols;
  a.dec = dec;
  a.dh = h / 2;
  a.dw = w / 2;
  memset(&tmap, 0, sizeof(tmap));
  static const bool no_tma = getenv("CT_NO_TMA") != nullptr;  // debugging switch: force the LDG loader
  a.use_tma = !no_tma && encode_tmap_2d(&tmap, frames, sizeof(T), (uint64_t)w,
                                        (uint64_t)(n_videos * n_frames * (int64_t)h), BC, BR + 1);
  return a.use_tma;
}

// Band partials of one level (no finalize).
template <typename T, int BC>
int launch_partials(const MomentArgs& a, const CUtensorMap& tmap, cudaStream_t st) {
  constexpr int BR = band_rows<T>();
  constexpr int NB = ring_buffers<T>();
  constexpr int CPT = cols_per_thread<T, BC>();
  const int n_chunks = (a.n_frames - 1 + a.chunk - 1) / a.chunk;
  CT_REQUIRE(a.n_videos <= 65535 && n_chunks <= 65535, "too many videos/chunks for one launch");
  dim3 grid((unsigned)a.units, (unsigned)n_chunks, (unsigned)a.n_videos);
  static const bool sync_kernel = getenv("CT_MOM_SYNC") != nullptr;  // probing: the CTA-barrier kernel
  if (a.use_tma && !sync_kernel) {
    constexpr int RS = row_split<T>();
    using S = SmemWS<T, BR, NB, BC, BC / CPT * RS>;
    auto kern = ttc_moments_ws_kernel<T, BR, NB, BC, CPT, RS>;
    CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::total));
    kern<<<grid, BC / CPT * RS, S::total, st>>>(a, tmap);
  } else {
    constexpr int CPS = cols_per_thread_sync<T, BC>();
    using S = Smem<T, BR, NB, BC, BC / CPS>;
    auto kern = ttc_moments_kernel<T, BR, NB, BC, CPS>;
    CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::total));
    kern<<<grid, BC / CPS, S::total, st>>>(a, tmap);
  }
  return check_launch("ttc_moments");
}

template <typename T, int BC>
int launch_bc(const T* frames, int64_t n_videos, int n_frames, int h, int w, int border, double* sums, void* ws,
              size_t ws_size, void* dec, cudaStream_t st) {
  const size_t need = ws_bytes<T>(n_videos, n_frames, h, w);
  CT_REQUIRE(ws != nullptr && ws_size >= need, "moments workspace too small (%zu < %zu)", ws_size, need);
  MomentArgs a;
  CUtensorMap tmap;
  prep_level<T, BC>(a, tmap, frames, n_videos, n_frames, h, w, border, reinterpret_cast<double*>(ws), dec);
  int rc = launch_partials<T, BC>(a, tmap, st);
  if (rc) return rc;
  const int64_t n_sys = n_videos * (n_frames - 1);
  const double count = (double)(h - 1 - 2 * border) * (double)(w - 1 - 2 * border);
  moments_finalize_kernel<<<finalize_grid(n_sys), kFinWarps * 32, 0, st>>>(a.partials, n_sys, a.units, count, sums);
  return check_launch("moments_finalize");
}

template <typename T>
int launch(const T* frames, int64_t n_videos, int n_frames, int h, int w, int border, double* sums, void* ws,
           size_t ws_size, void* dec, cudaStream_t st) {
  if (n_frames - 1 <= 0 || n_videos == 0) return CT_OK;
  if (pick_bc(w) == 128) return launch_bc<T, 128>(frames, n_videos, n_frames, h, w, border, sums, ws, ws_size, dec, st);
  return launch_bc<T, 256>(frames, n_videos, n_frames, h, w, border, sums, ws, ws_size, dec, st);
}

// Band partials of several levels: one launch of the levels kernel when every
// level has a TMA map, else one launch per level.
template <typename T, int BC>
int launch_levels_bc(const MomentLevel* lv, int n, int64_t n_videos, int n_frames, int border, cudaStream_t st) {
  CT_REQUIRE(n >= 1 && n <= kMaxLevels, "1..%d levels per launch", kMaxLevels);
  LevelsArgs m;
  memset(&m, 0, sizeof(m));
  m.n = n;
  bool all_tma = getenv("CT_MOM_SYNC") == nullptr;
  int64_t ctas = 0;
  for (int l = 0; l < n; ++l) {
    all_tma &= prep_level<T, BC>(m.a[l], m.tmap[l], reinterpret_cast<const T*>(lv[l].frames), n_videos, n_frames,
                                 lv[l].h, lv[l].w, border, lv[l].partials, lv[l].dec, lv[l].chunk);
    const int n_chunks = (n_frames - 1 + m.a[l].chunk - 1) / m.a[l].chunk;
    ctas += (int64_t)m.a[l].units * n_chunks * n_videos;
    m.cta_end[l] = ctas;
  }
  if (n == 1 || !all_tma || ctas > 0x7fffffffll) {
    for (int l = 0; l < n; ++l) {
      int rc = launch_partials<T, BC>(m.a[l], m.tmap[l], st);
      if (rc) return rc;
    }
    return CT_OK;
  }
  constexpr int BR = band_rows<T>();
  constexpr int NB = ring_buffers<T>();
  constexpr int CPT = cols_per_thread<T, BC>();
  constexpr int RS = row_split<T>();
  using S = SmemWS<T, BR, NB, BC, BC / CPT * RS>;
  auto kern = ttc_moments_levels_kernel<T, BR, NB, BC, CPT, RS>;
  CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::total));
  kern<<<(unsigned)ctas, BC / CPT * RS, S::total, st>>>(m);
  return check_launch("ttc_moments_levels");
}

}  // namespace

size_t moments_workspace(int dtype, int64_t n_videos, int n_frames, int h, int w) {
  return dtype == CT_F64 ? ws_bytes<double>(n_videos, n_frames, h, w) : ws_bytes<float>(n_videos, n_frames, h, w);
}

int moments_launch(int dtype, const void* frames, int64_t n_videos, int n_frames, int h, int w, int border,
                   double* sums, void* ws, size_t ws_size, cudaStream_t st, void* dec) {
  if (dtype == CT_F64)
    return launch<double>((const double*)frames, n_videos, n_frames, h, w, border, sums, ws, ws_size, dec, st);
  return launch<float>((const float*)frames, n_videos, n_frames, h, w, border, sums, ws, ws_size, dec, st);
}

int moments_units(int dtype, int64_t n_videos, int n_frames, int h, int w) {
  return dtype == CT_F64 ? make_plan<double>(n_videos, n_frames, h, w).units
                         : make_plan<float>(n_videos, n_frames, h, w).units;
}

int moments_levels_launch(int dtype, const MomentLevel* lv, int n_levels, int64_t n_videos, int n_frames, int border,
                          cudaStream_t st) {
  if (n_frames - 1 <= 0 || n_videos == 0 || n_levels == 0) return CT_OK;
  const int w0 = lv[0].w;
  if (dtype == CT_F64)
    return pick_bc(w0) == 128 ? launch_levels_bc<double, 128>(lv, n_levels, n_videos, n_frames, border, st)
                              : launch_levels_bc<double, 256>(lv, n_levels, n_videos, n_frames, border, st);
  return pick_bc(w0) == 128 ? launch_levels_bc<float, 128>(lv, n_levels, n_videos, n_frames, border, st)
                            : launch_levels_bc<float, 256>(lv, n_levels, n_videos, n_frames, border, st);
}

int partials_finalize(const double* partials, int64_t n_sys, int units, double count, double* sums,
                      cudaStream_t st) {
  if (n_sys == 0) return CT_OK;
  moments_finalize_kernel<<<finalize_grid(n_sys), kFinWarps * 32, 0, st>>>(partials, n_sys, units, count, sums);
  return check_launch("moments_finalize");
}

}  // namespace ct
