// Direct n-D correlation / convolution (K1-K4) for sm_100a.
//
// Replaces the reference's compiled loops _loops.xcorr_{valid,zpad}_{1,2,3}d
// and the numpy shift-and-add path for ndim >= 4 (_loops.py:27-208), behind
// the semantics layer conv._direct (conv.py:133-158).
//
// Per-output arithmetic is kept identical to the reference: taps are
// accumulated from 0.0 in row-major (j0, j1, j2) order with FMA for ranks 1-3
// (numba fastmath contracts `out += kv * s`), and with a rounded multiply
// followed by a rounded add for ranks >= 4 (numpy `out += k[idx] * s[win]`).
// Zero extension adds fma(k, 0, acc) == acc for taps the reference skips, so
// float64 results are bit-identical to the reference for finite inputs.
//
// Two kernels:
//  * xcorr_tiled<T, NW, VX, TY, TZ>: ranks 1-3.  A CTA stages a signal tile
//    (with the K-1 halo, zero- or clamp-filled) per input z-slice in shared
//    memory, each thread owns a TZ x TY x VX register block of outputs (VX
//    consecutive x, loaded as one 16-byte vector per chunk).  Input rows are
//    the outer loop so every staged value feeds up to TZ*TY*VX FMAs; kernel
//    taps live in the kernel-parameter constant bank (uniform operands).
//    NW (kernel x extent) is a compile-time parameter for the widths below.
//  * xcorr_strip<T>: ranks 1-3, any kernel width (runtime, strips of 8
//    compile-time taps, taps staged in shared memory): the widths without a
//    tiled instantiation.
//  * xcorr_generic<T>: any rank <= CT_MAXDIM and any kernel width; one thread
//    per output, odometer over taps.  Used for ranks >= 4 (and kernels too
//    large for the strip kernel's shared memory).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "tma.cuh"

namespace ct {
namespace {

constexpr int kMaxTapsF64 = 1024;  // 8 KB of kernel parameters
constexpr int kMaxTapsF32 = 2048;  // 8 KB

template <typename T>
struct MaxTaps;
template <>
struct MaxTaps<double> {
  static constexpr int value = kMaxTapsF64;
};
template <>
struct MaxTaps<float> {
  static constexpr int value = kMaxTapsF32;
};

template <typename T>
struct alignas(16) TapsParam {  // 16-byte aligned: tap rows load as 128-bit uniform loads
  T v[MaxTaps<T>::value];
};

template <typename T, int VX>
struct VecT;
template <>
struct VecT<double, 2> {
  using type = double2;
};
template <>
struct VecT<float, 4> {
  using type = float4;
};
struct alignas(16) Double4x2 {  // four doubles as two 16-byte vectors (no 32-byte shared-memory loads)
  double2 lo, hi;
};
struct alignas(16) Float4x2 {  // eight floats as two 16-byte vectors
  float4 lo, hi;
};
template <>
struct VecT<float, 8> {
  using type = Float4x2;
};
template <>
struct VecT<double, 4> {
  using type = Double4x2;
};

struct TileArgs {
  const void* s;
  void* out;
  int64_t batch;
  int mz, my, mx;
  int oz, oy, ox;
  int nz, ny;
  int pz, py, px;
  int boundary;
  int txn, tyn;  // threads along x, thread rows
  int tiles_z;   // z tiles per signal
  int sx, sy;    // staged tile extents (elements)
};

__device__ __forceinline__ double fmadd(double k, double v, double acc) { return fma(k, v, acc); }
__device__ __forceinline__ float fmadd(float k, float v, float acc) { return fmaf(k, v, acc); }

template <typename T, int NW, int VX, int TY, int TZ>
__global__ void __launch_bounds__(256) xcorr_tiled(const TileArgs a,
                                                   const __grid_constant__ TapsParam<T> taps) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tile = reinterpret_cast<T*>(smem_raw);
  using V = typename VecT<T, VX>::type;
  constexpr int CH = (VX + NW - 1 + VX - 1) / VX;  // vector chunks per input row window

  const int tid = threadIdx.x;
  const int nthr = blockDim.x;
  const int tx = tid % a.txn, ty = tid / a.txn;
  const int BX = a.txn * VX, BY = a.tyn * TY;
  const int x0 = blockIdx.x * BX, y0 = blockIdx.y * BY;
  const int ny = a.ny, nz = a.nz;
  const int64_t plane = (int64_t)a.my * a.mx;
  const int64_t n_ztiles = a.batch * a.tiles_z;

  for (int64_t bz = blockIdx.z; bz < n_ztiles; bz += gridDim.z) {
    const int64_t b = bz / a.tiles_z;
    const int z0 = (int)(bz % a.tiles_z) * TZ;
    const T* s = reinterpret_cast<const T*>(a.s) + b * (int64_t)a.mz * plane;

    T acc[TZ][TY][VX];
#pragma unroll
    for (int i = 0; i < TZ; ++i)
#pragma unroll
      for (int j = 0; j < TY; ++j)
#pragma unroll
        for (int r = 0; r < VX; ++r) acc[i][j][r] = T(0);

    const int nzin = TZ + nz - 1;
    for (int izr = 0; izr < nzin; ++izr) {
      int gz = z0 - a.pz + izr;
      if (gz < 0 || gz >= a.mz) {
        if (a.boundary == CT_ZERO) continue;  // all-zero slice: adds nothing
        gz = gz < 0 ? 0 : a.mz - 1;
      }
      __syncthreads();  // previous slice fully consumed
      {
        const T* sp = s + gz * plane;
        const int iy0 = y0 - a.py, ix0 = x0 - a.px;
        const int total = a.sx * a.sy;
        for (int idx = tid; idx < total; idx += nthr) {
          const int r = idx / a.sx, c = idx - r * a.sx;
          int gy = iy0 + r, gx = ix0 + c;
          T v = T(0);
          const bool in = (unsigned)gy < (unsigned)a.my && (unsigned)gx < (unsigned)a.mx;
          if (in) {
            v = __ldg(sp + (int64_t)gy * a.mx + gx);
          } else if (a.boundary == CT_REPLICATE) {
            gy = min(max(gy, 0), a.my - 1);
            gx = min(max(gx, 0), a.mx - 1);
            v = __ldg(sp + (int64_t)gy * a.mx + gx);
          }
          tile[idx] = v;
        }
      }
      __syncthreads();

      const int nrows = TY + ny - 1;
      for (int r = 0; r < nrows; ++r) {
        // every thread-row window value of this staged input row
        T v[CH * VX];
        const T* rowp = tile + (ty * TY + r) * a.sx + tx * VX;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const V q = *reinterpret_cast<const V*>(rowp + c * VX);
          const T* qp = reinterpret_cast<const T*>(&q);
#pragma unroll
          for (int e = 0; e < VX; ++e) v[c * VX + e] = qp[e];
        }
#pragma unroll
        for (int zi = 0; zi < TZ; ++zi) {
          const int j0 = izr - zi;
          if (j0 < 0 || j0 >= nz) continue;
#pragma unroll
          for (int yi = 0; yi < TY; ++yi) {
            const int j1 = r - yi;
            if (j1 < 0 || j1 >= ny) continue;
            const T* kr = taps.v + (j0 * ny + j1) * NW;
#pragma unroll
            for (int j2 = 0; j2 < NW; ++j2) {
              const T kv = kr[j2];
#pragma unroll
              for (int rr = 0; rr < VX; ++rr) acc[zi][yi][rr] = fmadd(kv, v[rr + j2], acc[zi][yi][rr]);
            }
          }
        }
      }
    }

    // store the register block
    T* out = reinterpret_cast<T*>(a.out) + b * (int64_t)a.oz * a.oy * a.ox;
#pragma unroll
    for (int zi = 0; zi < TZ; ++zi) {
      const int z = z0 + zi;
      if (z >= a.oz) break;
#pragma unroll
      for (int yi = 0; yi < TY; ++yi) {
        const int y = y0 + ty * TY + yi;
        if (y >= a.oy) break;
        T* orow = out + ((int64_t)z * a.oy + y) * a.ox;
        const int x = x0 + tx * VX;
#pragma unroll
        for (int rr = 0; rr < VX; ++rr)
          if (x + rr < a.ox) orow[x + rr] = acc[zi][yi][rr];
      }
    }
  }
}

struct GenArgs {
  const void* s;
  const void* k;
  void* out;
  int64_t batch;
  int ndim;
  int boundary;
  int fused;
  int flip;
  int64_t ms[CT_MAXDIM], ns[CT_MAXDIM], pl[CT_MAXDIM], os[CT_MAXDIM];
  int64_t sstr[CT_MAXDIM];
  int64_t s_elems, o_elems, k_elems;
};

template <typename T>
__device__ __forceinline__ T mul_add_rn(T k, T v, T acc);
template <>
__device__ __forceinline__ double mul_add_rn(double k, double v, double acc) {
  return __dadd_rn(acc, __dmul_rn(k, v));
}
template <>
__device__ __forceinline__ float mul_add_rn(float k, float v, float acc) {
  return __fadd_rn(acc, __fmul_rn(k, v));
}

template <typename T>
__global__ void __launch_bounds__(256) xcorr_generic(const GenArgs a) {
  const int64_t total = a.batch * a.o_elems;
  const T* kk = reinterpret_cast<const T*>(a.k);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / a.o_elems;
    int64_t rem = i - b * a.o_elems;
    int64_t o[CT_MAXDIM];
    for (int d = a.ndim - 1; d >= 0; --d) {
      o[d] = rem % a.os[d];
      rem /= a.os[d];
    }
    const T* s = reinterpret_cast<const T*>(a.s) + b * a.s_elems;
    T acc = T(0);
    int64_t j[CT_MAXDIM];
    for (int d = 0; d < a.ndim; ++d) j[d] = 0;
    for (int64_t t = 0; t < a.k_elems; ++t) {
      int64_t off = 0;
      bool in = true;
      for (int d = 0; d < a.ndim; ++d) {
        int64_t si = o[d] - a.pl[d] + j[d];
        if (si < 0 || si >= a.ms[d]) {
          if (a.boundary == CT_ZERO) {
            in = false;
            break;
          }
          si = si < 0 ? 0 : a.ms[d] - 1;
        }
        off += si * a.sstr[d];
      }
      if (in) {
        const T kv = kk[a.flip ? a.k_elems - 1 - t : t];
        const T sv = s[off];
        acc = a.fused ? fmadd(kv, sv, acc) : mul_add_rn(kv, sv, acc);
      }
      for (int d = a.ndim - 1; d >= 0; --d) {  // odometer, row-major
        if (++j[d] < a.ns[d]) break;
        j[d] = 0;
      }
    }
    reinterpret_cast<T*>(a.out)[i] = acc;
  }
}

// ---------------------------------------------------------------------------
// Width-generic register-tiled correlation (ranks 1-3, any kernel width): the
// xcorr_tiled schedule with the kernel's x extent a runtime value.  The taps
// are staged once per CTA into shared memory (flip applied, every kernel row
// padded to a multiple of C), the x taps run as strips of C compile-time
// taps (a runtime loop over full strips plus one compile-time tail strip of
// nw % C taps, so no padded tap is ever multiplied), and per staged input row
// a thread loads its VX + C - 1 window values of a strip once and reuses them
// for its TY x TZ output rows.  Per output the taps are applied in row-major
// (j0, j1, j2) order from 0.0 (strips in order), so fp64 results are
// bit-identical to the reference loops (_loops.py:104-198).
template <typename T, int W, int C, int VX, int TY, int TZ, bool ALLY = false>
__device__ __forceinline__ void strip_fma(const T* __restrict__ rowp, const T* __restrict__ taps, int nwp,
                                          int izr, int r, int nz, int ny, T (&acc)[TZ][TY][VX]) {
  using V = typename VecT<T, VX>::type;
  constexpr int CH = (VX + W - 1 + VX - 1) / VX;
  T v[CH * VX];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const V q = *reinterpret_cast<const V*>(rowp + c * VX);
    const T* qp = reinterpret_cast<const T*>(&q);
#pragma unroll
    for (int e = 0; e < VX; ++e) v[c * VX + e] = qp[e];
  }
#pragma unroll
  for (int zi = 0; zi < TZ; ++zi) {
    const int j0 = izr - zi;
    if (j0 < 0 || j0 >= nz) continue;
#pragma unroll
    for (int yi = 0; yi < TY; ++yi) {
      const int j1 = r - yi;
      if (!ALLY && (j1 < 0 || j1 >= ny)) continue;  // ALLY: TY - 1 <= r < ny, every output row takes this input row
      const T* kr = taps + (j0 * ny + j1) * nwp;  // uniform address: constant-bank or broadcast loads
      T kv[(W + VX - 1) / VX * VX];  // 16-byte vector loads (rows are padded to kStripC taps)
#pragma unroll
      for (int q = 0; q < (W + VX - 1) / VX; ++q) {
        const V t = *reinterpret_cast<const V*>(kr + q * VX);
        const T* tp = reinterpret_cast<const T*>(&t);
#pragma unroll
        for (int e = 0; e < VX; ++e) kv[q * VX + e] = tp[e];
      }
#pragma unroll
      for (int j2 = 0; j2 < W; ++j2)
#pragma unroll
        for (int rr = 0; rr < VX; ++rr) acc[zi][yi][rr] = fmadd(kv[j2], v[rr + j2], acc[zi][yi][rr]);
    }
  }
}

// PARAM: the (flipped, row-padded) taps come in the kernel-parameter bank
// (uniform constant loads, no shared-memory traffic: 13x13 fp64 10.9 -> 13.2
// TFLOP/s against taps in shared memory), else they are staged from the device kernel
// into shared memory (kernels larger than the 8 KB bank, graph capture
// without a host copy of the kernel).
template <typename T, int C, int VX, int TY, int TZ, bool PARAM>
__global__ void __launch_bounds__(256) xcorr_strip(const TileArgs a, const T* __restrict__ k, int nw, int flip,
                                                   const __grid_constant__ TapsParam<T> tp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nwp = (nw + C - 1) / C * C;  // padded taps per kernel row
  const int nrow_k = a.nz * a.ny;
  T* taps_smem = reinterpret_cast<T*>(smem_raw);
  T* tile = PARAM ? taps_smem : taps_smem + ((size_t)nrow_k * nwp + 3) / 4 * 4;  // 16-byte aligned after the taps
  const T* taps = PARAM ? tp.v : taps_smem;
  const int tid = threadIdx.x, nthr = blockDim.x;
  if (!PARAM) {
    const int64_t kt = (int64_t)nrow_k * nw;
    for (int idx = tid; idx < nrow_k * nwp; idx += nthr) {
      const int row = idx / nwp, j2 = idx - row * nwp;
      const int64_t t = (int64_t)row * nw + j2;
      taps_smem[idx] = j2 < nw ? __ldg(k + (flip ? kt - 1 - t : t)) : T(0);  // padding is never multiplied
    }
  }
  const int tx = tid % a.txn, ty = tid / a.txn;
  const int BX = a.txn * VX, BY = a.tyn * TY;
  const int x0 = blockIdx.x * BX, y0 = blockIdx.y * BY;
  const int ny = a.ny, nz = a.nz;
  const int64_t plane = (int64_t)a.my * a.mx;
  const int64_t n_ztiles = a.batch * a.tiles_z;
  const int full = nw / C, tail = nw - full * C;

  for (int64_t bz = blockIdx.z; bz < n_ztiles; bz += gridDim.z) {
    const int64_t b = bz / a.tiles_z;
    const int z0 = (int)(bz % a.tiles_z) * TZ;
    const T* s = reinterpret_cast<const T*>(a.s) + b * (int64_t)a.mz * plane;
    T acc[TZ][TY][VX];
#pragma unroll
    for (int i = 0; i < TZ; ++i)
#pragma unroll
      for (int j = 0; j < TY; ++j)
#pragma unroll
        for (int r = 0; r < VX; ++r) acc[i][j][r] = T(0);
    const int nzin = TZ + nz - 1;
    for (int izr = 0; izr < nzin; ++izr) {
      int gz = z0 - a.pz + izr;
      if (gz < 0 || gz >= a.mz) {
        if (a.boundary == CT_ZERO) continue;  // all-zero slice: adds nothing
        gz = gz < 0 ? 0 : a.mz - 1;
      }
      __syncthreads();  // previous slice consumed (and the taps staged, first time)
      {
        // staged tile, one warp per row (no index division per element)
        const T* sp = s + gz * plane;
        const int iy0 = y0 - a.py, ix0 = x0 - a.px;
        const int lane = tid & 31, nwarp = nthr >> 5;
        for (int r = tid >> 5; r < a.sy; r += nwarp) {
          int gy = iy0 + r;
          const bool row_in = (unsigned)gy < (unsigned)a.my;
          if (!row_in && a.boundary == CT_REPLICATE) gy = min(max(gy, 0), a.my - 1);
          const T* srow = sp + (int64_t)gy * a.mx;
          T* trow = tile + r * a.sx;
          for (int c = lane; c < a.sx; c += 32) {
            int gx = ix0 + c;
            T v = T(0);
            if (row_in && (unsigned)gx < (unsigned)a.mx) {
              v = __ldg(srow + gx);
            } else if (a.boundary == CT_REPLICATE) {
              gx = min(max(gx, 0), a.mx - 1);
              v = __ldg(srow + gx);
            }
            trow[c] = v;
          }
        }
      }
      __syncthreads();
      const int nrows = TY + ny - 1;
      for (int r = 0; r < nrows; ++r) {
        const T* rowp = tile + (ty * TY + r) * a.sx + tx * VX;
        if (TZ == 1 && r >= TY - 1 && r < ny) {  // interior input row (2-D): no per-output-row test
          for (int st = 0; st < full; ++st)
            strip_fma<T, C, C, VX, TY, TZ, true>(rowp + st * C, taps + st * C, nwp, izr, r, nz, ny, acc);
        } else {
          for (int st = 0; st < full; ++st)
            strip_fma<T, C, C, VX, TY, TZ>(rowp + st * C, taps + st * C, nwp, izr, r, nz, ny, acc);
        }
        const T* rt = rowp + full * C;
        const T* kt_ = taps + full * C;
        const bool ally = TZ == 1 && r >= TY - 1 && r < ny;
        switch (tail) {  // compile-time tail strip
#define CT_TAIL(Wt)                                                                       \
  case Wt:                                                                                \
    if (ally)                                                                             \
      strip_fma<T, Wt, C, VX, TY, TZ, true>(rt, kt_, nwp, izr, r, nz, ny, acc);           \
    else                                                                                  \
      strip_fma<T, Wt, C, VX, TY, TZ>(rt, kt_, nwp, izr, r, nz, ny, acc);                 \
    break;
          CT_TAIL(1) CT_TAIL(2) CT_TAIL(3) CT_TAIL(4) CT_TAIL(5) CT_TAIL(6) CT_TAIL(7)
#undef CT_TAIL
          default: break;
        }
      }
    }
    T* out = reinterpret_cast<T*>(a.out) + b * (int64_t)a.oz * a.oy * a.ox;
#pragma unroll
    for (int zi = 0; zi < TZ; ++zi) {
      const int z = z0 + zi;
      if (z >= a.oz) break;
#pragma unroll
      for (int yi = 0; yi < TY; ++yi) {
        const int y = y0 + ty * TY + yi;
        if (y >= a.oy) break;
        T* orow = out + ((int64_t)z * a.oy + y) * a.ox;
        const int x = x0 + tx * VX;
#pragma unroll
        for (int rr = 0; rr < VX; ++rr)
          if (x + rr < a.ox) orow[x + rr] = acc[zi][yi][rr];
      }
    }
  }
}

#ifndef CT_STRIP_TY64
#define CT_STRIP_TY64 4
#endif
#ifndef CT_STRIP_VX64
#define CT_STRIP_VX64 2
#endif
#ifndef CT_STRIP_TY32
#define CT_STRIP_TY32 4
#endif
#ifndef CT_STRIP_VX32
#define CT_STRIP_VX32 8  // 33x33 fp32: 0.449 -> 0.423 ms against 4 columns per thread (one LDCU per 8 FFMAs)
#endif
constexpr int kStripC = 8;  // compile-time taps per strip (a multiple of both vector widths)
template <typename T>
constexpr int strip_vx() {  // outputs per thread along x
  return sizeof(T) == 8 ? CT_STRIP_VX64 : CT_STRIP_VX32;
}

inline void choose_tile(const TileArgs& a, int nw, int vx, int rows_per_thread, int* txn, int* tyn,
                        bool whole_warps);  // below: threads (txn x tyn) minimising padded outputs + staging

// smem bytes of xcorr_strip for these extents (0: does not fit one CTA)
template <typename T>
size_t strip_smem(const TileArgs& a, int nw, int txn, int tyn, int TY, bool param = false) {
  constexpr int VX = strip_vx<T>();
  const int nwp = (nw + kStripC - 1) / kStripC * kStripC;
  const size_t taps = param ? 0 : ((size_t)a.nz * a.ny * nwp + 3) / 4 * 4;
  const int BX = txn * VX, BY = tyn * TY;
  const int sx = BX - VX + (VX + nwp - 1 + VX - 1) / VX * VX;  // every strip's window loads stay in the row
  const size_t tile = (size_t)sx * (BY + a.ny - 1);
  const size_t bytes = (taps + tile) * sizeof(T);
  return bytes <= 200 * 1024 ? bytes : 0;
}

template <typename T, int TY, int TZ>
int launch_strip(const TileArgs& a0, const T* k_dev, const T* taps_host, int nw, int flip, cudaStream_t st) {
  constexpr int VX = strip_vx<T>();
  TileArgs a = a0;
  a.txn = 32;
  a.tyn = 8;
  const int nwp = (nw + kStripC - 1) / kStripC * kStripC;
  // taps_host: the flipped taps in row-major order (nullptr: stage from k_dev)
  const bool param = taps_host != nullptr && (int64_t)a.nz * a.ny * nwp <= MaxTaps<T>::value;
  {  // thread block shape fitted to the output extents (268^2 outputs: 25 % padded with 32 x 8 threads)
    int tx = 32, ty = 8;
    choose_tile(a, nwp, VX, TY, &tx, &ty, false);
    const size_t fit = strip_smem<T>(a, nw, tx, ty, TY, param);
    if (fit > 0 && fit <= 64 * 1024 && getenv("CT_STRIP_FIXED_TILE") == nullptr) {
      a.txn = tx;
      a.tyn = ty;
    }
  }
  const size_t smem = strip_smem<T>(a, nw, a.txn, a.tyn, TY, param);
  CT_REQUIRE(smem > 0, "kernel too large for the strip kernel");
  a.sx = a.txn * VX - VX + (VX + nwp - 1 + VX - 1) / VX * VX;
  a.sy = a.tyn * TY + a.ny - 1;
  a.tiles_z = TZ > 1 ? (int)cdiv(a.oz, TZ) : a.oz;
  TapsParam<T> tp;
  if (param)
    for (int row = 0; row < a.nz * a.ny; ++row)
      for (int j2 = 0; j2 < nwp; ++j2) tp.v[row * nwp + j2] = j2 < nw ? taps_host[row * nw + j2] : T(0);
  auto kern = param ? xcorr_strip<T, kStripC, VX, TY, TZ, true> : xcorr_strip<T, kStripC, VX, TY, TZ, false>;
  CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)cdiv(a.ox, a.txn * VX), (unsigned)cdiv(a.oy, a.tyn * TY),
            (unsigned)std::min<int64_t>(a.batch * a.tiles_z, 65535));
  kern<<<grid, a.txn * a.tyn, smem, st>>>(a, k_dev, nw, flip, tp);
  return check_launch("xcorr_strip");
}

// Tile walk of the persistent 2-D kernels: tile t = (image b, tile row, tile
// column) advanced by a fixed step (the grid size) with carries instead of two
// integer divisions per tile (the division sequences, executed by every thread
// for the output addresses, were ~15 % of the cfg1 kernel's warp samples).
struct TileWalk {
  int b, ty, tx;     // current tile
  int sb, sy, sx;    // the step in mixed radix (tiles_x, tiles_y)
  int tiles_x, tiles_y;
  __device__ __forceinline__ void init(int64_t t, int64_t step, int tiles_x_, int tiles_y_) {
    tiles_x = tiles_x_;
    tiles_y = tiles_y_;
    const int64_t per = (int64_t)tiles_x * tiles_y;
    b = (int)(t / per);
    int r = (int)(t - (int64_t)b * per);
    ty = r / tiles_x;
    tx = r - ty * tiles_x;
    sb = (int)(step / per);
    r = (int)(step - (int64_t)sb * per);
    sy = r / tiles_x;
    sx = r - sy * tiles_x;
  }
  __device__ __forceinline__ void next() {
    tx += sx;
    const int cx = tx >= tiles_x;
    tx -= cx ? tiles_x : 0;
    ty += sy + cx;
    const int cy = ty >= tiles_y;
    ty -= cy ? tiles_y : 0;
    b += sb + cy;
  }
};

// ---------------------------------------------------------------------------
// 2-D zero-extended correlation with TMA-staged tiles (the HBM-bound small-
// kernel case, BASELINE config 1).  Persistent CTAs walk output tiles of the
// whole batch; each tile's input window (BY+NH-1 rows x SX columns, starting
// at (x0-px, y0-py)) is one cp.async.bulk.tensor box whose out-of-range
// elements the TMA unit zero-fills -- exactly the FULL/SAME zero padding, with
// no per-element index math.  Two smem stages: the next tile streams in while
// the current one is computed.  Compute is the xcorr_tiled register block
// (TY rows x VX columns per thread, row-major FMA tap order: bit-identical).
// outputs per thread along x in the TMA kernel: one 16-byte vector (measured:
// 4 doubles per thread is 20% slower than 2 on config 1)
template <typename T>
constexpr int tma_vx() { return 16 / sizeof(T); }

#ifndef CT_TMA2D_STAGES
#define CT_TMA2D_STAGES 2
#endif
constexpr int kTma2dStages = CT_TMA2D_STAGES;  // TMA ring depth of the 2-D conv kernel

template <typename T, int NW, int VX, int TY, int NH>
__global__ void __launch_bounds__(256) xcorr_tma2d(const TileArgs a, const __grid_constant__ TapsParam<T> taps,
                                                   const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) unsigned char smem_tma[];
  constexpr int VW = 16 / sizeof(T);  // elements per 16-byte vector; VX is a multiple of it
  using V = typename VecT<T, VW>::type;
  constexpr int CH = (VX + NW - 1 + VX - 1) / VX;
  const int tid = threadIdx.x;
  const int tx = tid % a.txn, ty = tid / a.txn;
  const int BX = a.txn * VX, BY = a.tyn * TY;
  const int tiles_x = (a.ox + BX - 1) / BX, tiles_y = (a.oy + BY - 1) / BY;
  const int64_t n_tiles = (int64_t)tiles_x * tiles_y * a.batch;
  const size_t stage_bytes = ((size_t)a.sx * a.sy * sizeof(T) + 127) & ~size_t(127);
  auto stage = [&](int s) { return reinterpret_cast<T*>(smem_tma + (size_t)s * stage_bytes); };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_tma + kTma2dStages * stage_bytes);
  const uint32_t box_bytes = (uint32_t)(a.sx * a.sy * sizeof(T));
  const int ny = a.ny;

  auto issue = [&](const TileWalk& w, int s) {
    mbar_arrive_expect_tx(&bars[s], box_bytes);
    tma_load_3d(stage(s), &tmap, &bars[s], w.tx * BX - a.px, w.ty * BY - a.py, w.b);
  };
  if (tid == 0) {
    for (int k = 0; k < kTma2dStages; ++k) mbar_init(&bars[k], 1);
    mbar_fence_init();
  }
  __syncthreads();
  int64_t t = blockIdx.x;
  TileWalk cur, pre;  // the tile being computed / the tile kTma2dStages steps ahead (the refill)
  cur.init(t, gridDim.x, tiles_x, tiles_y);
  pre = cur;
  for (int k = 0; k < kTma2dStages; ++k) {
    if (tid == 0 && t + k * (int64_t)gridDim.x < n_tiles) issue(pre, k);
    pre.next();
  }
  // per-thread constants of the output addressing
  const int lx = tx * VX, ly = ty * TY;
  for (int it = 0; t < n_tiles; ++it, t += gridDim.x, cur.next(), pre.next()) {
    const int s = it % kTma2dStages;
    mbar_wait(&bars[s], (uint32_t)((it / kTma2dStages) & 1));
    const T* tile = stage(s);
    T acc[TY][VX];
#pragma unroll
    for (int j = 0; j < TY; ++j)
#pragma unroll
      for (int r = 0; r < VX; ++r) acc[j][r] = T(0);
    // NH > 0: kernel height known at compile time -> the row loop unrolls and
    // every tap index is a constant (taps become constant-bank operands)
    const int nrows = TY + (NH > 0 ? NH : ny) - 1;
#pragma unroll
    for (int r = 0; r < (NH > 0 ? TY + NH - 1 : nrows); ++r) {
      T v[CH * VX];
      const T* rowp = tile + (ty * TY + r) * a.sx + tx * VX;
#pragma unroll
      for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int k = 0; k < VX / VW; ++k) {
          const V q = *reinterpret_cast<const V*>(rowp + c * VX + k * VW);
          const T* qp = reinterpret_cast<const T*>(&q);
#pragma unroll
          for (int e = 0; e < VW; ++e) v[c * VX + k * VW + e] = qp[e];
        }
#pragma unroll
      for (int yi = 0; yi < TY; ++yi) {
        const int j1 = r - yi;
        if (j1 < 0 || j1 >= (NH > 0 ? NH : ny)) continue;
        const T* kr = taps.v + j1 * NW;
#pragma unroll
        for (int j2 = 0; j2 < NW; ++j2) {
          const T kv = kr[j2];
#pragma unroll
          for (int rr = 0; rr < VX; ++rr) acc[yi][rr] = fmadd(kv, v[rr + j2], acc[yi][rr]);
        }
      }
    }
    __syncthreads();  // stage s fully read: refill it with the tile kTma2dStages steps ahead
    if (tid == 0 && t + kTma2dStages * (int64_t)gridDim.x < n_tiles) {
      fence_proxy_async_smem();
      issue(pre, s);
    }
    const int x = cur.tx * BX + lx, y = cur.ty * BY + ly;
    T* orow = reinterpret_cast<T*>(a.out) + ((int64_t)cur.b * a.oy + y) * a.ox + x;
    const int rows = a.oy - y;  // output rows of this thread that exist (<= 0: none)
    const bool vec_store = (a.ox % VW == 0) && (x + VX <= a.ox);
#pragma unroll
    for (int yi = 0; yi < TY; ++yi) {
      if (yi >= rows) break;
      if (vec_store) {
#pragma unroll
        for (int k = 0; k < VX / VW; ++k) {
          V q;
          T* qp = reinterpret_cast<T*>(&q);
#pragma unroll
          for (int e = 0; e < VW; ++e) qp[e] = acc[yi][k * VW + e];
          *reinterpret_cast<V*>(orow + k * VW) = q;
        }
      } else {
#pragma unroll
        for (int rr = 0; rr < VX; ++rr)
          if (x + rr < a.ox) orow[rr] = acc[yi][rr];
      }
      orow += a.ox;
    }
  }
}

template <typename T, int NW, int VX, int TY, int NH>
int launch_tma2d(const TileArgs& a0, const T* taps_host, int ntaps, cudaStream_t st) {
  TileArgs a = a0;
  TapsParam<T> taps;
  for (int i = 0; i < ntaps; ++i) taps.v[i] = taps_host[i];
  const int BX = a.txn * VX, BY = a.tyn * TY;
  constexpr int CH = (VX + NW - 1 + VX - 1) / VX;
  a.sx = BX - VX + CH * VX;
  a.sy = BY + a.ny - 1;
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  if (!encode_tmap_3d(&tmap, a.s, sizeof(T), (uint64_t)a.mx, (uint64_t)a.my, (uint64_t)a.batch, a.sx, a.sy)) {
    set_error("tensor map encode failed");
    return CT_EUNSUPPORTED;
  }
  const size_t stage_bytes = ((size_t)a.sx * a.sy * sizeof(T) + 127) & ~size_t(127);
  const size_t smem = kTma2dStages * stage_bytes + 8 * kTma2dStages;
  auto kern = xcorr_tma2d<T, NW, VX, TY, NH>;
  CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, a.txn * a.tyn, smem));
  const int64_t tiles = cdiv(a.ox, BX) * cdiv(a.oy, BY) * a.batch;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)num_sms() * std::max(1, per_sm)));
  kern<<<grid, a.txn * a.tyn, smem, st>>>(a, taps, tmap);
  return check_launch("xcorr_tma2d");
}

// Width-generic 2-D correlation with TMA-staged tiles: xcorr_tma2d's
// persistent tile walk and 2-stage ring (zero extension by TMA fill, the next
// tile in flight during the FMAs) with xcorr_strip's runtime-width compute
// (taps in the parameter bank, strips of C compile-time taps plus one
// compile-time tail).  Replaces the LDG-staged strip kernel where the box
// start is 16-byte aligned: its per-tile staging (every warp waiting on its
// global loads between two CTA barriers) was 24 % of the 13x13 fp64 kernel's
// warp time.  Same per-output tap order: fp64 bit-identical.
template <typename T, int C, int VX, int TY>
__global__ void __launch_bounds__(256) xcorr_tma2d_strip(const TileArgs a, const __grid_constant__ TapsParam<T> tp,
                                                         const __grid_constant__ CUtensorMap tmap, int nw) {
  extern __shared__ __align__(128) unsigned char smem_tms[];
  constexpr int VW = 16 / sizeof(T);
  using V = typename VecT<T, VW>::type;
  const int nwp = (nw + C - 1) / C * C;
  const int tid = threadIdx.x;
  const int tx = tid % a.txn, ty = tid / a.txn;
  const int BX = a.txn * VX, BY = a.tyn * TY;
  const int tiles_x = (a.ox + BX - 1) / BX, tiles_y = (a.oy + BY - 1) / BY;
  const int64_t n_tiles = (int64_t)tiles_x * tiles_y * a.batch;
  const size_t stage_bytes = ((size_t)a.sx * a.sy * sizeof(T) + 127) & ~size_t(127);
  auto stage = [&](int s) { return reinterpret_cast<T*>(smem_tms + (size_t)s * stage_bytes); };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_tms + 2 * stage_bytes);
  const uint32_t box_bytes = (uint32_t)(a.sx * a.sy * sizeof(T));
  const int ny = a.ny;
  const int full = nw / C, tail = nw - full * C;
  const T* taps = tp.v;

  auto issue = [&](const TileWalk& w, int s) {
    mbar_arrive_expect_tx(&bars[s], box_bytes);
    tma_load_3d(stage(s), &tmap, &bars[s], w.tx * BX - a.px, w.ty * BY - a.py, w.b);
  };
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  int64_t t = blockIdx.x;
  TileWalk cur, pre;  // the tile being computed / the tile two steps ahead (the refill)
  cur.init(t, gridDim.x, tiles_x, tiles_y);
  pre = cur;
  for (int k = 0; k < 2; ++k) {
    if (tid == 0 && t + k * (int64_t)gridDim.x < n_tiles) issue(pre, k);
    pre.next();
  }
  const int lx = tx * VX, ly = ty * TY;
  for (int it = 0; t < n_tiles; ++it, t += gridDim.x, cur.next(), pre.next()) {
    const int s = it & 1;
    mbar_wait(&bars[s], (uint32_t)((it >> 1) & 1));
    const T* tile = stage(s);
    T acc[1][TY][VX];
#pragma unroll
    for (int j = 0; j < TY; ++j)
#pragma unroll
      for (int r = 0; r < VX; ++r) acc[0][j][r] = T(0);
    const int nrows = TY + ny - 1;
    for (int r = 0; r < nrows; ++r) {
      const T* rowp = tile + (ty * TY + r) * a.sx + tx * VX;
      if (r >= TY - 1 && r < ny) {  // interior input row: no per-output-row test, one block of TY * C * VX FMAs
        for (int st = 0; st < full; ++st)
          strip_fma<T, C, C, VX, TY, 1, true>(rowp + st * C, taps + st * C, nwp, 0, r, 1, ny, acc);
      } else {
        for (int st = 0; st < full; ++st)
          strip_fma<T, C, C, VX, TY, 1>(rowp + st * C, taps + st * C, nwp, 0, r, 1, ny, acc);
      }
      const T* rt = rowp + full * C;
      const T* kt_ = taps + full * C;
      const bool ally = r >= TY - 1 && r < ny;
      switch (tail) {  // compile-time tail strip
#define CT_TAIL(Wt)                                                                   \
  case Wt:                                                                            \
    if (ally)                                                                         \
      strip_fma<T, Wt, C, VX, TY, 1, true>(rt, kt_, nwp, 0, r, 1, ny, acc);           \
    else                                                                              \
      strip_fma<T, Wt, C, VX, TY, 1>(rt, kt_, nwp, 0, r, 1, ny, acc);                 \
    break;
        CT_TAIL(1) CT_TAIL(2) CT_TAIL(3) CT_TAIL(4) CT_TAIL(5) CT_TAIL(6) CT_TAIL(7)
#undef CT_TAIL
        default: break;
      }
    }
    __syncthreads();  // stage s fully read: refill it with the tile two steps ahead
    if (tid == 0 && t + 2 * (int64_t)gridDim.x < n_tiles) {
      fence_proxy_async_smem();
      issue(pre, s);
    }
    const int x = cur.tx * BX + lx, y = cur.ty * BY + ly;
    T* orow = reinterpret_cast<T*>(a.out) + ((int64_t)cur.b * a.oy + y) * a.ox + x;
    const int rows = a.oy - y;
    const bool vec_store = (a.ox % VW == 0) && (x + VX <= a.ox);
#pragma unroll
    for (int yi = 0; yi < TY; ++yi) {
      if (yi >= rows) break;
      if (vec_store) {
#pragma unroll
        for (int k = 0; k < VX / VW; ++k) {
          V q;
          T* qp = reinterpret_cast<T*>(&q);
#pragma unroll
          for (int e = 0; e < VW; ++e) qp[e] = acc[0][yi][k * VW + e];
          *reinterpret_cast<V*>(orow + k * VW) = q;
        }
      } else {
#pragma unroll
        for (int rr = 0; rr < VX; ++rr)
          if (x + rr < a.ox) orow[rr] = acc[0][yi][rr];
      }
      orow += a.ox;
    }
  }
}

// CT_UNSUPPORTED-free probe: can the TMA strip kernel take this problem?
template <typename T>
bool tma_strip_ok(const TileArgs& a, int nw, bool have_host_taps) {
  const int nwp = (nw + kStripC - 1) / kStripC * kStripC;
  // kernels up to ~20 x 20 taps: beyond that a tile's FMAs dwarf its staging and the second stage only
  // costs occupancy (33x33 fp32: 0.57 ms with the ring against 0.45 ms for the LDG-staged kernel)
  return have_host_taps && a.oz == 1 && a.nz == 1 && a.mz == 1 && a.boundary == CT_ZERO &&
         (int64_t)a.ny * nwp <= 400 && (a.px * (int)sizeof(T)) % 16 == 0 &&
         (a.mx * (int64_t)sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(a.s) & 15) == 0 &&
         a.batch < (1ll << 31) && getenv("CT_CONV_NOTMA") == nullptr;
}

template <typename T, int TY>
int launch_tma2d_strip(const TileArgs& a0, const T* taps_host, int nw, cudaStream_t st) {
  constexpr int VX = strip_vx<T>();
  TileArgs a = a0;
  a.txn = 32;
  a.tyn = 8;
  const int nwp = (nw + kStripC - 1) / kStripC * kStripC;
  if (getenv("CT_STRIP_FIXED_TILE") == nullptr) choose_tile(a, nwp, VX, TY, &a.txn, &a.tyn, false);
  a.sx = a.txn * VX - VX + (VX + nwp - 1 + VX - 1) / VX * VX;
  a.sy = a.tyn * TY + a.ny - 1;
  const size_t stage_bytes = ((size_t)a.sx * a.sy * sizeof(T) + 127) & ~size_t(127);
  const size_t smem = 2 * stage_bytes + 16;
  // two stages above 64 KB cost more occupancy than the overlap returns (33x33 fp32: 0.545 vs 0.458 ms
  // for the LDG-staged kernel): the caller falls back
  if (a.sx > 256 || a.sy > 256 || smem > 64 * 1024) return CT_EUNSUPPORTED;
  TapsParam<T> tp;
  for (int row = 0; row < a.ny; ++row)
    for (int j2 = 0; j2 < nwp; ++j2) tp.v[row * nwp + j2] = j2 < nw ? taps_host[row * nw + j2] : T(0);
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  if (!encode_tmap_3d(&tmap, a.s, sizeof(T), (uint64_t)a.mx, (uint64_t)a.my, (uint64_t)a.batch, a.sx, a.sy))
    return CT_EUNSUPPORTED;
  auto kern = xcorr_tma2d_strip<T, kStripC, VX, TY>;
  CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, a.txn * a.tyn, smem));
  const int64_t tiles = cdiv(a.ox, a.txn * VX) * cdiv(a.oy, a.tyn * TY) * a.batch;
  const unsigned grid =
      (unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)num_sms() * std::max(1, per_sm)));
  kern<<<grid, a.txn * a.tyn, smem, st>>>(a, tp, tmap, nw);
  return check_launch("xcorr_tma2d_strip");
}

template <typename T, int LW>
struct LoadT;
template <>
struct LoadT<float, 4> {
  using type = float4;
};
template <>
struct LoadT<float, 2> {
  using type = float2;
};
template <>
struct LoadT<float, 1> {
  using type = float;
};
template <>
struct LoadT<double, 2> {
  using type = double2;
};
template <>
struct LoadT<double, 1> {
  using type = double;
};

// ---------------------------------------------------------------------------
// 3-D zero-extended correlation with TMA-staged z-slices (BASELINE config 3).
// A CTA owns TZ output slices x (BY x BX) of one volume and walks the input
// slices that feed them through a 2-stage TMA ring (4-D tensor map
// {x, y, z, batch}: out-of-range slices, rows and columns arrive as zeros).
// The box starts at x0 - pxa with pxa = px rounded up to a 16-byte multiple,
// so the window of thread tx begins `sh` = pxa - px elements into its staged
// row; LW (elements per shared load: 4, 2 or 1) keeps those loads aligned.
template <typename T, int NW, int VX, int TY, int TZ, int LW>
__global__ void __launch_bounds__(256) xcorr_tma3d(const TileArgs a, const __grid_constant__ TapsParam<T> taps,
                                                   const __grid_constant__ CUtensorMap tmap, int pxa) {
  extern __shared__ __align__(128) unsigned char smem_tma[];
  constexpr int CHL = (VX + NW - 1 + LW - 1) / LW;  // window loads per row
  using L = typename LoadT<T, LW>::type;
  const int tid = threadIdx.x;
  const int tx = tid % a.txn, ty = tid / a.txn;
  const int BX = a.txn * VX, BY = a.tyn * TY;
  const int x0 = blockIdx.x * BX, y0 = blockIdx.y * BY;
  const int sh = pxa - a.px;
  const size_t stage_bytes = ((size_t)a.sx * a.sy * sizeof(T) + 127) & ~size_t(127);
  auto stage = [&](int s) { return reinterpret_cast<T*>(smem_tma + (size_t)s * stage_bytes); };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_tma + 2 * stage_bytes);
  const uint32_t box_bytes = (uint32_t)(a.sx * a.sy * sizeof(T));
  const int ny = a.ny, nz = a.nz;
  const int64_t n_ztiles = a.batch * a.tiles_z;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  int gcount = 0;  // slices this CTA has consumed so far: stage = g & 1, phase = (g >> 1) & 1
  for (int64_t bz = blockIdx.z; bz < n_ztiles; bz += gridDim.z) {
    const int b = (int)(bz / a.tiles_z);
    const int z0 = (int)(bz % a.tiles_z) * TZ;
    // input slices gz in [z0 - pz, z0 - pz + TZ + nz - 1) that exist
    const int g_lo = max(0, z0 - a.pz), g_hi = min(a.mz, z0 - a.pz + TZ + nz - 1);
    const int nsl = max(0, g_hi - g_lo);
    const int g0 = gcount;
    auto issue = [&](int k) {  // k-th existing slice -> stage (g0 + k) & 1
      if (tid == 0) {
        const int sg = (g0 + k) & 1;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bars[sg], box_bytes);
        tma_load_4d(stage(sg), &tmap, &bars[sg], x0 - pxa, y0 - a.py, g_lo + k, b);
      }
    };
    if (nsl > 0) issue(0);
    if (nsl > 1) issue(1);
    T acc[TZ][TY][VX];
#pragma unroll
    for (int i = 0; i < TZ; ++i)
#pragma unroll
      for (int j = 0; j < TY; ++j)
#pragma unroll
        for (int r = 0; r < VX; ++r) acc[i][j][r] = T(0);
    for (int k = 0; k < nsl; ++k) {
      const int g = g0 + k;
      const int s = g & 1;
      mbar_wait(&bars[s], (uint32_t)((g >> 1) & 1));
      const T* tile = stage(s);
      const int izr = g_lo + k - (z0 - a.pz);  // slice index relative to the window start
      const int nrows = TY + ny - 1;
      for (int r = 0; r < nrows; ++r) {
        T v[CHL * LW];
        const T* rowp = tile + (ty * TY + r) * a.sx + sh + tx * VX;
#pragma unroll
        for (int c = 0; c < CHL; ++c) {
          const L q = *reinterpret_cast<const L*>(rowp + c * LW);
          const T* qp = reinterpret_cast<const T*>(&q);
#pragma unroll
          for (int e = 0; e < LW; ++e) v[c * LW + e] = qp[e];
        }
#pragma unroll
        for (int zi = 0; zi < TZ; ++zi) {
          const int j0 = izr - zi;
          if (j0 < 0 || j0 >= nz) continue;
#pragma unroll
          for (int yi = 0; yi < TY; ++yi) {
            const int j1 = r - yi;
            if (j1 < 0 || j1 >= ny) continue;
            const T* kr = taps.v + (j0 * ny + j1) * NW;
#pragma unroll
            for (int j2 = 0; j2 < NW; ++j2) {
              const T kv = kr[j2];
#pragma unroll
              for (int rr = 0; rr < VX; ++rr) acc[zi][yi][rr] = fmadd(kv, v[rr + j2], acc[zi][yi][rr]);
            }
          }
        }
      }
      __syncthreads();  // stage s consumed
      if (k + 2 < nsl) issue(k + 2);
    }
    gcount += nsl;
    T* out = reinterpret_cast<T*>(a.out) + (int64_t)b * a.oz * a.oy * a.ox;
#pragma unroll
    for (int zi = 0; zi < TZ; ++zi) {
      const int z = z0 + zi;
      if (z >= a.oz) break;
#pragma unroll
      for (int yi = 0; yi < TY; ++yi) {
        const int y = y0 + ty * TY + yi;
        if (y >= a.oy) break;
        T* orow = out + ((int64_t)z * a.oy + y) * a.ox;
        const int x = x0 + tx * VX;
#pragma unroll
        for (int rr = 0; rr < VX; ++rr)
          if (x + rr < a.ox) orow[x + rr] = acc[zi][yi][rr];
      }
    }
  }
}

template <typename T, int NW, int VX, int TY, int TZ>
int launch_tma3d(const TileArgs& a0, const T* taps_host, int ntaps, cudaStream_t st) {
  TileArgs a = a0;
  TapsParam<T> taps;
  for (int i = 0; i < ntaps; ++i) taps.v[i] = taps_host[i];
  constexpr int VW = 16 / sizeof(T);
  const int pxa = (a.px + VW - 1) / VW * VW;
  const int sh = pxa - a.px;
  const int BX = a.txn * VX, BY = a.tyn * TY;
  a.sx = sh + BX + NW - 1;
  a.sx = (a.sx + VW - 1) / VW * VW;  // 16-byte box rows
  a.sy = BY + a.ny - 1;
  a.tiles_z = (int)cdiv(a.oz, TZ);
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  if (!encode_tmap_4d(&tmap, a.s, sizeof(T), (uint64_t)a.mx, (uint64_t)a.my, (uint64_t)a.mz, (uint64_t)a.batch, a.sx,
                      a.sy)) {
    set_error("tensor map encode failed");
    return CT_EUNSUPPORTED;
  }
  const size_t stage_bytes = ((size_t)a.sx * a.sy * sizeof(T) + 127) & ~size_t(127);
  const size_t smem = 2 * stage_bytes + 16 + 16;  // + barriers; window over-read of <= 12 bytes stays inside
  dim3 grid((unsigned)cdiv(a.ox, BX), (unsigned)cdiv(a.oy, BY),
            (unsigned)std::min<int64_t>(a.batch * a.tiles_z, 65535));
  int rc;
  if (sh % 4 == 0 && VW == 4) {
    auto kern = xcorr_tma3d<T, NW, VX, TY, TZ, (VW == 4 ? 4 : 2)>;
    CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, a.txn * a.tyn, smem, st>>>(a, taps, tmap, pxa);
  } else if (sh % 2 == 0) {
    auto kern = xcorr_tma3d<T, NW, VX, TY, TZ, 2>;
    CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, a.txn * a.tyn, smem, st>>>(a, taps, tmap, pxa);
  } else {
    auto kern = xcorr_tma3d<T, NW, VX, TY, TZ, 1>;
    CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, a.txn * a.tyn, smem, st>>>(a, taps, tmap, pxa);
  }
  rc = check_launch("xcorr_tma3d");
  return rc;
}

// ---------------------------------------------------------------------------
// 3-D z-walking correlation (large 3-D kernels, BASELINE config 3).
// Work item = one output slice of one (BY x BX) output column block.  The
// kernel is persistent: CTA c takes items [c*per_cta, (c+1)*per_cta) of the
// flattened (volume, tile row, tile column, z) order, i.e. one or two runs of
// consecutive output slices, so every SM gets the same number of slices.
// For a run [z0, z1) the CTA streams the input z-slices that feed it through
// a TMA ring (4-D map, zero-filled halos).  Every staged slice s is used by
// all NZ kernel planes at once: register slot j holds output z = s + pz - j,
// so slot j accumulates plane j of the kernel from this slice; after the
// slice, slot NZ-1 is complete (stored) and the slots shift by one.  Kernel
// indices (j0 = slot, j2) are compile-time and j1 is a short loop, so the
// taps come from the parameter bank with a uniform offset, and each staged
// value feeds NZ * TY * NW FMAs.  Per output the taps are still applied in
// row-major (j0, j1, j2) order from 0.0, so fp64 results are bit-exact.
// Work split of the z-walking kernels.  nc > 0: every (volume, tile) column is
// cut into nc runs of consecutive output slices [zb[i], zb[i+1]) of equal
// WORK -- an output slice costs one kernel plane per input slice that exists,
// so the first and last NZ-1 slices of a FULL-mode column are cheaper -- and
// CTA c takes run c % nc of column c / nc: one run per CTA (one pipeline
// fill), no run straddling two columns.  nc == 0: the flattened (column, z)
// slices in equal counts per CTA (more columns than CTA slots).
constexpr int kMaxZRuns = 32;
struct ZRuns {
  int nc;
  int zb[kMaxZRuns + 1];
};

inline ZRuns plan_zruns(const TileArgs& a, int nz, int64_t columns, int64_t slots) {
  ZRuns r;
  memset(&r, 0, sizeof(r));
  if (getenv("CT_ZW_FLAT")) return r;  // probing only
  int64_t nc = columns > 0 ? slots / columns : 0;
  nc = std::min<int64_t>(nc, std::min<int64_t>(kMaxZRuns, a.oz / (2 * nz)));
  if (nc < 1 || (double)(nc * columns) < 0.9 * (double)slots) return r;
  std::vector<int64_t> pre(a.oz + 1, 0);  // work prefix: planes with an existing input slice
  for (int z = 0; z < a.oz; ++z) {
    const int lo = std::max(0, z - a.pz), hi = std::min(a.mz, z - a.pz + nz);
    pre[z + 1] = pre[z] + std::max(0, hi - lo) + 1;  // + 1: the per-slice store / bookkeeping
  }
  r.nc = (int)nc;
  int z = 0;
  for (int i = 1; i < nc; ++i) {
    const double target = (double)pre[a.oz] * i / (double)nc;
    while (z < a.oz && (double)pre[z + 1] <= target) ++z;
    // the nearer of pre[z], pre[z + 1]
    if (z < a.oz && target - (double)pre[z] > (double)pre[z + 1] - target) ++z;
    r.zb[i] = std::max(z, r.zb[i - 1] + 1);
  }
  r.zb[nc] = a.oz;
  for (int i = (int)nc - 1; i > 0; --i) r.zb[i] = std::min(r.zb[i], r.zb[i + 1] - 1);
  return r;
}

#ifndef CT_ZW_WARP_REL
#define CT_ZW_WARP_REL 1  // per-warp stage release (0: CTA barrier per slice, the round-1 kernel)
#endif
template <typename T, int NZ, int NH, int NW, int TY, int VX, int LW, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) xcorr_zwalk(const TileArgs a, const __grid_constant__ TapsParam<T> taps,
                                                      const __grid_constant__ CUtensorMap tmap, int pxa,
                                                      int64_t per_cta, const __grid_constant__ ZRuns zr) {
  extern __shared__ __align__(128) unsigned char smem_zw[];
  constexpr int NS = 3;                             // TMA ring stages
  constexpr int CW = VX + NW - 1;                   // window columns per row
  constexpr int CHL = (CW + LW - 1) / LW;           // loads per window row
  constexpr int KP = (NW * sizeof(T) + 15) / 16 * 16 / sizeof(T);  // padded taps per kernel row
  using L = typename LoadT<T, LW>::type;
  const int tid = threadIdx.x;
  const int tx = tid % a.txn, ty = tid / a.txn;
  const int BX = a.txn * VX, BY = a.tyn * TY;
  const int tiles_x = (a.ox + BX - 1) / BX, tiles_y = (a.oy + BY - 1) / BY;
  const int sh = pxa - a.px;
  const size_t stage_bytes = ((size_t)a.sx * a.sy * sizeof(T) + 127) & ~size_t(127);
  auto stage = [&](int s) { return reinterpret_cast<T*>(smem_zw + (size_t)s * stage_bytes); };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_zw + NS * stage_bytes);
#if CT_ZW_WARP_REL
  int* rel = reinterpret_cast<int*>(smem_zw + NS * stage_bytes + 8 * NS);  // per-stage release counters
  const int nwarps = (int)(blockDim.x >> 5), lane = tid & 31;
#endif
  const uint32_t box_bytes = (uint32_t)(a.sx * a.sy * sizeof(T));
  const bool active = ty < a.tyn;
  const int64_t total = a.batch * tiles_y * tiles_x * (int64_t)a.oz;
  int64_t pos = (int64_t)blockIdx.x * per_cta;
  int64_t end = min(total, pos + per_cta);
  if (zr.nc > 0) {  // run blockIdx.x % nc of column blockIdx.x / nc
    const int64_t c0 = (int64_t)(blockIdx.x / zr.nc) * a.oz;
    pos = c0 + zr.zb[blockIdx.x % zr.nc];
    end = c0 + zr.zb[blockIdx.x % zr.nc + 1];
  }
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&bars[i], 1);
#if CT_ZW_WARP_REL
    for (int i = 0; i < NS; ++i) rel[i] = 0;
#endif
    mbar_fence_init();
  }
  __syncthreads();
  int gcount = 0;  // slices consumed by this CTA: ring stage g % NS, phase (g / NS) & 1

  while (pos < end) {
    const int64_t col = pos / a.oz;
    const int z0 = (int)(pos - col * a.oz);
    const int64_t left = end - pos;
    const int z1 = left < (int64_t)(a.oz - z0) ? z0 + (int)left : a.oz;
    pos += z1 - z0;
    const int b = (int)(col / (tiles_x * tiles_y));
    const int tt = (int)(col - (int64_t)b * tiles_x * tiles_y);
    const int x0 = (tt % tiles_x) * BX, y0 = (tt / tiles_x) * BY;
    // walk slices s in [z0 - pz, z1 - 1 - pz + NZ - 1]; real ones are [g_lo, g_hi)
    const int s_beg = z0 - a.pz, s_end = z1 - a.pz + NZ - 1;
    const int g_lo = max(0, s_beg), g_hi = min(a.mz, s_end);
    const int nsl = max(0, g_hi - g_lo);
    const int g0 = gcount;
    auto issue = [&](int k, bool any = false) {
      if (any || tid == 0) {
        const int st = (g0 + k) % NS;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bars[st], box_bytes);
        tma_load_4d(stage(st), &tmap, &bars[st], x0 - pxa, y0 - a.py, g_lo + k, b);
      }
    };
    for (int k = 0; k < NS && k < nsl; ++k) issue(k);

    T acc[NZ][TY][VX];
#pragma unroll
    for (int j = 0; j < NZ; ++j)
#pragma unroll
      for (int yi = 0; yi < TY; ++yi)
#pragma unroll
        for (int x = 0; x < VX; ++x) acc[j][yi][x] = T(0);

    T* out = reinterpret_cast<T*>(a.out) + (int64_t)b * a.oz * a.oy * a.ox;
    const int ox = x0 + tx * VX;
    for (int s = s_beg; s < s_end; ++s) {
      if (s >= g_lo && s < g_hi) {
        const int k = s - g_lo;
        const int g = g0 + k;
        mbar_wait(&bars[g % NS], (uint32_t)((g / NS) & 1));
        // slot j is live for this run when its output z = s + pz - j is in [z0, z1)
        const int jlo = max(0, s + a.pz - z1 + 1), jhi = min(NZ - 1, s + a.pz - z0);
        const T* tile = stage(g % NS) + (ty * TY) * a.sx + sh + tx * VX;
        if (active) {
#pragma unroll 1
          for (int j1 = 0; j1 < NH; ++j1) {
            T v[TY][CHL * LW];
#pragma unroll
            for (int yi = 0; yi < TY; ++yi) {
              const T* rp = tile + (yi + j1) * a.sx;
#pragma unroll
              for (int c = 0; c < CHL; ++c) {
                const L q = *reinterpret_cast<const L*>(rp + c * LW);
                const T* qp = reinterpret_cast<const T*>(&q);
#pragma unroll
                for (int e = 0; e < LW; ++e) v[yi][c * LW + e] = qp[e];
              }
            }
            // taps padded to KP per kernel row: 16-byte groups load as one uniform vector
            const T* kj1 = taps.v + j1 * KP;
            auto plane = [&](int j) {
              using V16 = typename LoadT<T, 16 / sizeof(T)>::type;
              constexpr int G = 16 / sizeof(T);
              T kr[KP];
#pragma unroll
              for (int q = 0; q < KP; q += G)
                *reinterpret_cast<V16*>(kr + q) = *reinterpret_cast<const V16*>(kj1 + j * NH * KP + q);
#pragma unroll
              for (int j2 = 0; j2 < NW; ++j2) {
                const T kv = kr[j2];
#pragma unroll
                for (int yi = 0; yi < TY; ++yi)
#pragma unroll
                  for (int x = 0; x < VX; ++x) acc[j][yi][x] = fmadd(kv, v[yi][x + j2], acc[j][yi][x]);
              }
            };
            if (jlo == 0 && jhi == NZ - 1) {  // interior slice: branch-free, all slots interleavable
#pragma unroll
              for (int j = 0; j < NZ; ++j) plane(j);
            } else {
#pragma unroll
              for (int j = 0; j < NZ; ++j)
                if (j >= jlo && j <= jhi) plane(j);
            }
          }
        }
#if CT_ZW_WARP_REL
        // stage consumed by this warp: the last warp to release it refills
        // it (no CTA barrier per slice; warps drift by up to NS - 1 slices)
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          if ((atomicAdd(&rel[g % NS], 1) % nwarps) == nwarps - 1 && k + NS < nsl) issue(k + NS, true);
        }
#else
        __syncthreads();  // stage consumed
        if (k + NS < nsl) issue(k + NS);
#endif
      }
      // slot NZ-1 now holds output z = s + pz - (NZ-1), complete
      const int zo = s + a.pz - (NZ - 1);
      if (zo >= z0 && zo < z1 && active) {
#pragma unroll
        for (int yi = 0; yi < TY; ++yi) {
          const int y = y0 + ty * TY + yi;
          if (y >= a.oy) break;
          T* orow = out + ((int64_t)zo * a.oy + y) * a.ox;
#pragma unroll
          for (int x = 0; x < VX; ++x)
            if (ox + x < a.ox) orow[ox + x] = acc[NZ - 1][yi][x];
        }
      }
#pragma unroll
      for (int j = NZ - 1; j > 0; --j)
#pragma unroll
        for (int yi = 0; yi < TY; ++yi)
#pragma unroll
          for (int x = 0; x < VX; ++x) acc[j][yi][x] = acc[j - 1][yi][x];
#pragma unroll
      for (int yi = 0; yi < TY; ++yi)
#pragma unroll
        for (int x = 0; x < VX; ++x) acc[0][yi][x] = T(0);
    }
    gcount += nsl;
#if CT_ZW_WARP_REL
    __syncthreads();  // run boundary: every stage free before the next run's first loads
#endif
  }
}

// Output tile for the z-walking kernel: threads txn x tyn (<= 256) minimising
// padded outputs plus staged halo over the (oy, ox) plane.
inline void choose_zwalk_tile(int oy, int ox, int vx, int ty_rows, int nh, int nw, int* txn, int* tyn,
                              int maxt = 256) {
  double best = 1e300;
  for (int tx = 16; tx <= 64; ++tx) {  // >= 16: a warp spans at most two staged rows (conflict-free LDS)
    for (int ty = 1; tx * ty <= maxt; ++ty) {
      if (tx * ty < maxt / 2) continue;
      const int bx = tx * vx, by = ty * ty_rows;
      if (bx + nw + 8 > 256 || by + nh - 1 > 256) continue;
      const double tiles = (double)cdiv(ox, bx) * (double)cdiv(oy, by);
      const double warps = (double)cdiv(tx * ty, 32) * 32;
      const double cost = tiles * (warps * vx * ty_rows * (double)nh * nw + 2.0 * (bx + nw) * (by + nh));
      if (cost < best * 0.999) {
        best = cost;
        *txn = tx;
        *tyn = ty;
      }
    }
  }
}

template <typename T, int NZ, int NH, int NW, int TY, int VX, int MAXT = 256>
int launch_zwalk(const TileArgs& a0, const T* taps_host, int ntaps, int zc_hint, cudaStream_t st) {
  TileArgs a = a0;
  constexpr int KP = (NW * sizeof(T) + 15) / 16 * 16 / sizeof(T);
  static_assert(NZ * NH * KP <= MaxTaps<T>::value, "padded taps exceed the parameter block");
  TapsParam<T> taps;
  for (int r = 0; r < NZ * NH; ++r)
    for (int j2 = 0; j2 < KP; ++j2) taps.v[r * KP + j2] = j2 < NW ? taps_host[r * NW + j2] : T(0);
  (void)ntaps;
  constexpr int VW = 16 / sizeof(T);
  if (a.txn <= 0 || a.tyn <= 0 || a.txn * a.tyn > MAXT) choose_zwalk_tile(a.oy, a.ox, VX, TY, NH, NW, &a.txn, &a.tyn, MAXT);
  if (getenv("CT_ZW_TXN") && getenv("CT_ZW_TYN")) {  // probing only
    a.txn = atoi(getenv("CT_ZW_TXN"));
    a.tyn = atoi(getenv("CT_ZW_TYN"));
  }
  const int pxa = (a.px + VW - 1) / VW * VW;
  const int sh = pxa - a.px;
  const int BX = a.txn * VX, BY = a.tyn * TY;
  a.sx = (sh + BX + NW - 1 + VW - 1) / VW * VW;
  a.sy = BY + NH - 1;
  const size_t stage_bytes = ((size_t)a.sx * a.sy * sizeof(T) + 127) & ~size_t(127);
  const size_t smem = 3 * stage_bytes + 64;
  CT_REQUIRE(smem <= 227 * 1024, "zwalk tile too large");
  const int nthr = (int)cdiv(a.txn * a.tyn, 32) * 32;
  void (*kern)(const TileArgs, const TapsParam<T>, const CUtensorMap, int, int64_t, const ZRuns);
  if (VW == 4 && sh % 4 == 0 && VX % 4 == 0)
    kern = xcorr_zwalk<T, NZ, NH, NW, TY, VX, (VW == 4 ? 4 : 2), MAXT>;
  else if (sh % 2 == 0)
    kern = xcorr_zwalk<T, NZ, NH, NW, TY, VX, 2, MAXT>;
  else
    kern = xcorr_zwalk<T, NZ, NH, NW, TY, VX, 1, MAXT>;
  CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 1;
  CT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nthr, smem));
  // persistent: the flattened (volume, tile, z) output slices split evenly
  // over every resident CTA slot (runs shorter than 2 NZ slices waste staging)
  const int64_t total = cdiv(a.ox, BX) * cdiv(a.oy, BY) * a.batch * a.oz;
  const int64_t slots = (int64_t)num_sms() * std::max(1, per_sm);
  int64_t per_cta = std::max<int64_t>(cdiv(total, slots), 2 * NZ);
  if (zc_hint > 0) per_cta = zc_hint;
  ZRuns zr = plan_zruns(a, NZ, total / a.oz, slots);
  if (zc_hint > 0) zr.nc = 0;
  if (const char* e = getenv("CT_ZW_ZC")) {  // probing only
    per_cta = std::max(1, atoi(e));
    zr.nc = 0;
  }
  const int64_t nctas = zr.nc > 0 ? (total / a.oz) * zr.nc : cdiv(total, per_cta);
  CT_REQUIRE(nctas < (1ll << 31), "too many z-walk CTAs");
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  if (a.sx > 256 || a.sy > 256 ||
      !encode_tmap_4d(&tmap, a.s, sizeof(T), (uint64_t)a.mx, (uint64_t)a.my, (uint64_t)a.mz, (uint64_t)a.batch, a.sx,
                      a.sy)) {
    set_error("tensor map encode failed");
    return CT_EUNSUPPORTED;
  }
  if (getenv("CT_DEBUG"))
    fprintf(stderr, "xcorr_zwalk TY %d MAXT %d: tile %dx%d (%d thr) per_cta %lld runs/column %d per_sm %d ctas %lld smem %zu\n",
            TY, MAXT, BX, BY, nthr, (long long)per_cta, zr.nc, per_sm, (long long)nctas, smem);
  kern<<<(unsigned)nctas, nthr, smem, st>>>(a, taps, tmap, pxa, per_cta, zr);
  return check_launch("xcorr_zwalk");
}

template <typename T, int NW, int VX, int TY, int TZ>
int launch_tiled(const TileArgs& a0, const T* k_host_order_taps, int ntaps, cudaStream_t st) {
  TileArgs a = a0;
  TapsParam<T> taps;
  for (int i = 0; i < ntaps; ++i) taps.v[i] = k_host_order_taps[i];
  const int BX = a.txn * VX, BY = a.tyn * TY;
  constexpr int CH = (VX + NW - 1 + VX - 1) / VX;
  a.sx = BX - VX + CH * VX;
  a.sy = BY + a.ny - 1;
  const size_t smem = (size_t)a.sx * a.sy * sizeof(T);
  auto kern = xcorr_tiled<T, NW, VX, TY, TZ>;
  if (smem > 48 * 1024) CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)cdiv(a.ox, BX), (unsigned)cdiv(a.oy, BY),
            (unsigned)std::min<int64_t>(a.batch * a.tiles_z, 65535));
  kern<<<grid, a.txn * a.tyn, smem, st>>>(a, taps);
  return check_launch("xcorr_tiled");
}

// ---------------------------------------------------------------------------
// fp32 row-pair kernel (K2/K3): packed f32x2 FMAs (FFMA2) on pairs of output
// rows.  Output rows y and y+1 use the same tap k[j0][j1][j2] on input rows
// y+j1 and y+1+j1, so the staged tile is kept as two row-pair interleaved
// copies (E: rows (2p, 2p+1), O: rows (2p+1, 2p+2)); every (row r, row r+1)
// column pair is then one aligned float2, the accumulators are (row, row+1)
// float2 pairs, and the taps are (k, k) pairs in the parameter bank, so one
// FFMA2 with a uniform-register tap does two output FMAs.  A thread owns
// TZ x 2 x 8 outputs (8 consecutive columns); per (slice, tap row) it loads
// its 8+NW-1 column window once and issues 8*NW FFMA2 per z output.
constexpr int kPairVX = 8;

struct TapsPairParam {
  float2 v[MaxTaps<float>::value];
};

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}

// Staged pair rows insert 2 padding float2 after every 8 logical columns, so
// thread tx's window starts at physical float2 10*tx: the eight lanes of a
// quarter-warp then hit eight different 16-byte bank groups, and the window
// chunk offsets 10*tx + 2c + 2*(c>>2) are compile-time per chunk.
__host__ __device__ __forceinline__ int pair_pad(int c) { return c + ((c >> 3) << 1); }

template <int NW, int TZ>
__global__ void __launch_bounds__(256) xcorr_pair_f32(const TileArgs a, const __grid_constant__ TapsPairParam taps) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int WIN = kPairVX + NW - 1;     // window columns (float2 pairs)
  constexpr int WLD = (WIN + 1) / 2;        // float4 loads per window
  const int tid = threadIdx.x;
  const int tx = tid % a.txn, ty = tid / a.txn;
  const int BX = a.txn * kPairVX, BY = a.tyn * 2;
  const int x0 = blockIdx.x * BX, y0 = blockIdx.y * BY;
  const int ny = a.ny, nz = a.nz;
  const int SY = a.sy, SXp = a.sx;          // staged rows, physical pitch (float2) of each pair copy
  const int SXl = BX - kPairVX + 2 * WLD;   // logical staged columns (every thread's window)
  const int PE = (SY + 1) / 2;              // pair rows in copy E
  float2* cE = reinterpret_cast<float2*>(smem_raw);
  float2* cO = cE + (size_t)PE * SXp;
  const int64_t plane = (int64_t)a.my * a.mx;
  const int64_t n_ztiles = a.batch * a.tiles_z;

  for (int64_t bz = blockIdx.z; bz < n_ztiles; bz += gridDim.z) {
    const int64_t b = bz / a.tiles_z;
    const int z0 = (int)(bz % a.tiles_z) * TZ;
    const float* s = reinterpret_cast<const float*>(a.s) + b * (int64_t)a.mz * plane;
    float2 acc[TZ][kPairVX];
#pragma unroll
    for (int i = 0; i < TZ; ++i)
#pragma unroll
      for (int m = 0; m < kPairVX; ++m) acc[i][m] = make_float2(0.f, 0.f);

    const int nzin = TZ + nz - 1;
    for (int izr = 0; izr < nzin; ++izr) {
      int gz = z0 - a.pz + izr;
      if (gz < 0 || gz >= a.mz) {
        if (a.boundary == CT_ZERO) continue;  // all-zero slice adds nothing
        gz = gz < 0 ? 0 : a.mz - 1;
      }
      __syncthreads();
      {
        const float* sp = s + gz * plane;
        const int iy0 = y0 - a.py, ix0 = x0 - a.px;
        float* fE = reinterpret_cast<float*>(cE);
        float* fO = reinterpret_cast<float*>(cO);
        // one warp per staged row, lanes along the (logical) columns
        const int lane = tid & 31, nwarps = blockDim.x >> 5;
        for (int r = tid >> 5; r < SY; r += nwarps) {
          int gy = iy0 + r;
          const bool row_in = (unsigned)gy < (unsigned)a.my;
          if (!row_in && a.boundary == CT_REPLICATE) gy = gy < 0 ? 0 : a.my - 1;
          const float* srow = sp + (int64_t)gy * a.mx;
          float* dE = fE + (size_t)(r >> 1) * SXp * 2 + (r & 1);
          float* dO = r >= 1 ? fO + (size_t)((r - 1) >> 1) * SXp * 2 + ((r - 1) & 1) : nullptr;
          for (int c = lane; c < SXl; c += 32) {
            int gx = ix0 + c;
            float v = 0.f;
            if (row_in && (unsigned)gx < (unsigned)a.mx) {
              v = __ldg(srow + gx);
            } else if (a.boundary == CT_REPLICATE) {
              gx = min(max(gx, 0), a.mx - 1);
              v = __ldg(srow + gx);
            }
            const int cp = pair_pad(c) * 2;
            dE[cp] = v;
            if (dO) dO[cp] = v;
          }
        }
        // the last pair row of each copy may reference a row past SY: zero it
        if (SY & 1) {
          for (int c = tid; c < SXp; c += blockDim.x) fE[(((SY - 1) >> 1) * SXp + c) * 2 + 1] = 0.f;
        } else {
          for (int c = tid; c < SXp; c += blockDim.x) fO[(((SY - 2) >> 1) * SXp + c) * 2 + 1] = 0.f;
        }
      }
      __syncthreads();

      for (int j1 = 0; j1 < ny; ++j1) {
        const int lr = 2 * ty + j1;  // local input row of the pair (lr, lr+1)
        const float2* prow = ((lr & 1) ? cO : cE) + (size_t)(lr >> 1) * SXp;
        float2 w[2 * WLD];
#pragma unroll
        for (int c = 0; c < WLD; ++c) {
          const float4 q = *reinterpret_cast<const float4*>(prow + 10 * tx + 2 * c + 2 * (c >> 2));
          w[2 * c] = make_float2(q.x, q.y);
          w[2 * c + 1] = make_float2(q.z, q.w);
        }
#pragma unroll
        for (int zi = 0; zi < TZ; ++zi) {
          const int j0 = izr - zi;
          if (j0 < 0 || j0 >= nz) continue;
          const float2* kr = taps.v + (j0 * ny + j1) * NW;
#pragma unroll
          for (int j2 = 0; j2 < NW; ++j2) {
            const float2 kk = kr[j2];
#pragma unroll
            for (int m = 0; m < kPairVX; ++m) acc[zi][m] = ffma2(kk, w[m + j2], acc[zi][m]);
          }
        }
      }
    }

    float* out = reinterpret_cast<float*>(a.out) + b * (int64_t)a.oz * a.oy * a.ox;
#pragma unroll
    for (int zi = 0; zi < TZ; ++zi) {
      const int z = z0 + zi;
      if (z >= a.oz) break;
      const int y = y0 + 2 * ty;
      const int x = x0 + tx * kPairVX;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (y + h >= a.oy) break;
        float* orow = out + ((int64_t)z * a.oy + y + h) * a.ox;
#pragma unroll
        for (int m = 0; m < kPairVX; ++m)
          if (x + m < a.ox) orow[x + m] = h ? acc[zi][m].y : acc[zi][m].x;
      }
    }
  }
}

template <int NW, int TZ>
int launch_pair_f32(const TileArgs& a0, const float* taps_host, int ntaps, cudaStream_t st) {
  TileArgs a = a0;
  TapsPairParam taps;
  for (int i = 0; i < ntaps; ++i) taps.v[i] = make_float2(taps_host[i], taps_host[i]);
  const int BX = a.txn * kPairVX, BY = a.tyn * 2;
  constexpr int WIN = kPairVX + NW - 1;
  constexpr int WLD = (WIN + 1) / 2;
  a.sy = BY + a.ny - 1;
  const int sxl = BX - kPairVX + 2 * WLD;  // logical columns covering every thread's window
  a.sx = pair_pad(sxl - 1) + 1;            // physical pitch with the bank-spreading padding
  a.sx += (a.sx & 1);                      // rows stay 16-byte aligned
  const int PE = (a.sy + 1) / 2, PO = a.sy / 2;
  const size_t smem = (size_t)(PE + PO) * a.sx * sizeof(float2);
  auto kern = xcorr_pair_f32<NW, TZ>;
  if (smem > 48 * 1024) CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)cdiv(a.ox, BX), (unsigned)cdiv(a.oy, BY),
            (unsigned)std::min<int64_t>(a.batch * a.tiles_z, 65535));
  kern<<<grid, a.txn * a.tyn, smem, st>>>(a, taps);
  return check_launch("xcorr_pair_f32");
}

// fp32 z-walking kernel with packed FFMA2 (same schedule as xcorr_zwalk:
// persistent runs of output slices, 3-stage TMA slice ring, NZ register
// slots).  The accumulators are (x, x+1) float2 pairs and the taps (k, k)
// pairs in the parameter bank (padded to 16 bytes per kernel row), so one
// FFMA2 does two output FMAs.  A window row is loaded as 16-byte vectors
// from the aligned base below it (SH4 = its offset, compile-time); the
// operand pairs (v[e], v[e+1]) are register pairs, odd ones built by moves.
template <int NZ, int NH, int NW, int TY, int SH4, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) xcorr_zwalk_x2(const TileArgs a, const __grid_constant__ TapsPairParam taps,
                                                         const __grid_constant__ CUtensorMap tmap, int pxa,
                                                         int64_t per_cta) {
  extern __shared__ __align__(128) unsigned char smem_zw2[];
  constexpr int NS = 3;
  constexpr int VX = 4;
  constexpr int NV4 = (SH4 + VX + NW - 1 + 3) / 4;  // 16-byte loads per window row
  constexpr int KP = (NW + 1) / 2 * 2;             // (k,k) pairs per kernel row, 16-byte padded
  const int tid = threadIdx.x;
  const int tx = tid % a.txn, ty = tid / a.txn;
  const int BX = a.txn * VX, BY = a.tyn * TY;
  const int tiles_x = (a.ox + BX - 1) / BX, tiles_y = (a.oy + BY - 1) / BY;
  const int sh = pxa - a.px;
  const size_t stage_bytes = ((size_t)a.sx * a.sy * sizeof(float) + 127) & ~size_t(127);
  auto stage = [&](int s) { return reinterpret_cast<float*>(smem_zw2 + (size_t)s * stage_bytes); };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_zw2 + NS * stage_bytes);
  const uint32_t box_bytes = (uint32_t)(a.sx * a.sy * sizeof(float));
  const bool active = ty < a.tyn;
  const int64_t total = a.batch * tiles_y * tiles_x * (int64_t)a.oz;
  int64_t pos = (int64_t)blockIdx.x * per_cta;
  const int64_t end = min(total, pos + per_cta);
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&bars[i], 1);
    mbar_fence_init();
  }
  __syncthreads();
  int gcount = 0;
  // aligned window base of this thread within a staged row (sh + tx*VX - SH4)
  const int wb = (ty * TY) * a.sx + sh + tx * VX - SH4;

  while (pos < end) {
    const int64_t col = pos / a.oz;
    const int z0 = (int)(pos - col * a.oz);
    const int64_t left = end - pos;
    const int z1 = left < (int64_t)(a.oz - z0) ? z0 + (int)left : a.oz;
    pos += z1 - z0;
    const int b = (int)(col / (tiles_x * tiles_y));
    const int tt = (int)(col - (int64_t)b * tiles_x * tiles_y);
    const int x0 = (tt % tiles_x) * BX, y0 = (tt / tiles_x) * BY;
    const int s_beg = z0 - a.pz, s_end = z1 - a.pz + NZ - 1;
    const int g_lo = max(0, s_beg), g_hi = min(a.mz, s_end);
    const int nsl = max(0, g_hi - g_lo);
    const int g0 = gcount;
    auto issue = [&](int k) {
      if (tid == 0) {
        const int st = (g0 + k) % NS;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bars[st], box_bytes);
        tma_load_4d(stage(st), &tmap, &bars[st], x0 - pxa, y0 - a.py, g_lo + k, b);
      }
    };
    for (int k = 0; k < NS && k < nsl; ++k) issue(k);

    float2 acc[NZ][TY][VX / 2];
#pragma unroll
    for (int j = 0; j < NZ; ++j)
#pragma unroll
      for (int yi = 0; yi < TY; ++yi)
#pragma unroll
        for (int x = 0; x < VX / 2; ++x) acc[j][yi][x] = make_float2(0.f, 0.f);

    float* out = reinterpret_cast<float*>(a.out) + (int64_t)b * a.oz * a.oy * a.ox;
    const int ox = x0 + tx * VX;
    for (int s = s_beg; s < s_end; ++s) {
      if (s >= g_lo && s < g_hi) {
        const int k = s - g_lo;
        const int g = g0 + k;
        mbar_wait(&bars[g % NS], (uint32_t)((g / NS) & 1));
        const int jlo = max(0, s + a.pz - z1 + 1), jhi = min(NZ - 1, s + a.pz - z0);
        const float* tile = stage(g % NS) + wb;
        if (active) {
#pragma unroll 1
          for (int j1 = 0; j1 < NH; ++j1) {
            float v[TY][NV4 * 4];
#pragma unroll
            for (int yi = 0; yi < TY; ++yi) {
              const float4* rp = reinterpret_cast<const float4*>(tile + (yi + j1) * a.sx);
#pragma unroll
              for (int c = 0; c < NV4; ++c) {
                const float4 q = rp[c];
                v[yi][4 * c] = q.x;
                v[yi][4 * c + 1] = q.y;
                v[yi][4 * c + 2] = q.z;
                v[yi][4 * c + 3] = q.w;
              }
            }
            const float2* kj1 = taps.v + j1 * KP;
            auto plane = [&](int j) {
              const float2* kr = kj1 + j * NH * KP;
#pragma unroll
              for (int j2 = 0; j2 < NW; ++j2) {
                const float2 kk = kr[j2];
#pragma unroll
                for (int yi = 0; yi < TY; ++yi)
#pragma unroll
                  for (int xp = 0; xp < VX / 2; ++xp) {
                    const int e = SH4 + 2 * xp + j2;
                    acc[j][yi][xp] = ffma2(kk, make_float2(v[yi][e], v[yi][e + 1]), acc[j][yi][xp]);
                  }
              }
            };
            if (jlo == 0 && jhi == NZ - 1) {
#pragma unroll
              for (int j = 0; j < NZ; ++j) plane(j);
            } else {
#pragma unroll
              for (int j = 0; j < NZ; ++j)
                if (j >= jlo && j <= jhi) plane(j);
            }
          }
        }
        __syncthreads();  // stage consumed
        if (k + NS < nsl) issue(k + NS);
      }
      const int zo = s + a.pz - (NZ - 1);
      if (zo >= z0 && zo < z1 && active) {
#pragma unroll
        for (int yi = 0; yi < TY; ++yi) {
          const int y = y0 + ty * TY + yi;
          if (y >= a.oy) break;
          float* orow = out + ((int64_t)zo * a.oy + y) * a.ox;
#pragma unroll
          for (int xp = 0; xp < VX / 2; ++xp) {
            if (ox + 2 * xp < a.ox) orow[ox + 2 * xp] = acc[NZ - 1][yi][xp].x;
            if (ox + 2 * xp + 1 < a.ox) orow[ox + 2 * xp + 1] = acc[NZ - 1][yi][xp].y;
          }
        }
      }
#pragma unroll
      for (int j = NZ - 1; j > 0; --j)
#pragma unroll
        for (int yi = 0; yi < TY; ++yi)
#pragma unroll
          for (int x = 0; x < VX / 2; ++x) acc[j][yi][x] = acc[j - 1][yi][x];
#pragma unroll
      for (int yi = 0; yi < TY; ++yi)
#pragma unroll
        for (int x = 0; x < VX / 2; ++x) acc[0][yi][x] = make_float2(0.f, 0.f);
    }
    gcount += nsl;
  }
}

template <int NZ, int NH, int NW, int TY, int MAXT = 256>
int launch_zwalk_x2(const TileArgs& a0, const float* taps_host, int ntaps, cudaStream_t st) {
  TileArgs a = a0;
  constexpr int KP = (NW + 1) / 2 * 2;
  static_assert(NZ * NH * KP <= MaxTaps<float>::value, "padded taps exceed the parameter block");
  TapsPairParam taps;
  for (int r = 0; r < NZ * NH; ++r)
    for (int j2 = 0; j2 < KP; ++j2) {
      const float kv = j2 < NW ? taps_host[r * NW + j2] : 0.f;
      taps.v[r * KP + j2] = make_float2(kv, kv);
    }
  (void)ntaps;
  constexpr int VX = 4;
  if (a.txn <= 0 || a.tyn <= 0 || a.txn * a.tyn > MAXT) choose_zwalk_tile(a.oy, a.ox, VX, TY, NH, NW, &a.txn, &a.tyn, MAXT);
  if (getenv("CT_ZW_TXN") && getenv("CT_ZW_TYN")) {  // probing only
    a.txn = atoi(getenv("CT_ZW_TXN"));
    a.tyn = atoi(getenv("CT_ZW_TYN"));
  }
  const int pxa = (a.px + 3) / 4 * 4;
  const int sh = pxa - a.px;  // 0..3
  const int BX = a.txn * VX, BY = a.tyn * TY;
  const int nv4 = (sh + VX + NW - 1 + 3) / 4;
  a.sx = std::max((sh + BX + NW - 1 + 3) / 4 * 4, BX - VX + 4 * nv4);  // every thread's vector loads stay in the row
  a.sy = BY + NH - 1;
  const size_t stage_bytes = ((size_t)a.sx * a.sy * sizeof(float) + 127) & ~size_t(127);
  const size_t smem = 3 * stage_bytes + 64;
  CT_REQUIRE(smem <= 227 * 1024, "zwalk tile too large");
  const int nthr = (int)cdiv(a.txn * a.tyn, 32) * 32;
  void (*kern)(const TileArgs, const TapsPairParam, const CUtensorMap, int, int64_t);
  switch (sh) {
    case 0: kern = xcorr_zwalk_x2<NZ, NH, NW, TY, 0, MAXT>; break;
    case 1: kern = xcorr_zwalk_x2<NZ, NH, NW, TY, 1, MAXT>; break;
    case 2: kern = xcorr_zwalk_x2<NZ, NH, NW, TY, 2, MAXT>; break;
    default: kern = xcorr_zwalk_x2<NZ, NH, NW, TY, 3, MAXT>; break;
  }
  CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 1;
  CT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nthr, smem));
  const int64_t total = cdiv(a.ox, BX) * cdiv(a.oy, BY) * a.batch * a.oz;
  const int64_t slots = (int64_t)num_sms() * std::max(1, per_sm);
  int64_t per_cta = std::max<int64_t>(cdiv(total, slots), 2 * NZ);
  if (const char* e = getenv("CT_ZW_ZC")) per_cta = std::max(1, atoi(e));  // probing only
  const int64_t nctas = cdiv(total, per_cta);
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  if (a.sx > 256 || a.sy > 256 ||
      !encode_tmap_4d(&tmap, a.s, sizeof(float), (uint64_t)a.mx, (uint64_t)a.my, (uint64_t)a.mz, (uint64_t)a.batch,
                      a.sx, a.sy)) {
    set_error("tensor map encode failed");
    return CT_EUNSUPPORTED;
  }
  if (getenv("CT_DEBUG"))
    fprintf(stderr, "xcorr_zwalk_x2 TY %d MAXT %d: tile %dx%d (%d thr) per_cta %lld per_sm %d ctas %lld\n", TY, MAXT,
            BX, BY, nthr, (long long)per_cta, per_sm, (long long)nctas);
  kern<<<(unsigned)nctas, nthr, smem, st>>>(a, taps, tmap, pxa, per_cta);
  return check_launch("xcorr_zwalk_x2");
}

// fp32 z-walking kernel with FFMA2 over pairs of kernel PLANES (config 3).
// Same schedule as xcorr_zwalk (persistent runs of output slices, 3-stage TMA
// slice ring released per warp, one output row x 8 columns per thread), but the
// NZ register slots of a column are kept as float2 pairs of z-adjacent slots:
// one staged value v feeds slots (j, j+1) with taps (k[j], k[j+1]), which is
// exactly FFMA2's (scalar broadcast) x (packed pair from a uniform register
// pair) + (packed accumulator) form -- no operand pair is ever built by moves,
// the staged layout stays the plain TMA tile, and 7 planes cost 3 FFMA2 + 1
// FFMA issue slots instead of 7.  The slots advance by one per slice, so the
// pairing alternates: per column e[0..NZ] (NZ odd),
//   even slice: slot j = e[j];           pairs (e0,e1)(e2,e3).. take (k0,k1)(k2,k3)..,
//               e[NZ-1] takes k[NZ-1] alone and is complete afterwards;
//   odd slice:  slot j = e[j-1], slot 0 = e[NZ]; pairs take (k1,k2)(k3,k4)..,
//               e[NZ] takes k0 alone, e[NZ-2] is complete afterwards;
//   then e' = [0, e[NZ], e0, .., e[NZ-3], 0] (two pair moves per column per
//   two slices).
// The parameter bank holds both tap orders per (j1, j2).  Slices at the ends of
// a run (not every slot live) take a scalar path with per-slot predicates.
template <int NZ, int SH4, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) xcorr_zwalk_zp(const TileArgs a, const __grid_constant__ TapsParam<float> taps,
                                                         const __grid_constant__ CUtensorMap tmap, int pxa,
                                                         int64_t per_cta, const __grid_constant__ ZRuns zr) {
  static_assert(NZ % 2 == 1, "plane pairs need an odd plane count");
  extern __shared__ __align__(128) unsigned char smem_zp[];
  constexpr int NS = 3;
  constexpr int VX = 8, NH = NZ, NW = NZ;
  constexpr int NP = NZ / 2;                        // full pairs; P[NP] = (e[NZ-1], e[NZ])
  constexpr int EP = (NZ + 1 + 3) / 4 * 4;          // floats per tap row
  constexpr int NV4 = (SH4 + VX + NW - 1 + 3) / 4;  // 16-byte loads per window row
  const int tid = threadIdx.x;
  const int tx = tid % a.txn, ty = tid / a.txn;
  const int BX = a.txn * VX, BY = a.tyn;
  const int tiles_x = (a.ox + BX - 1) / BX, tiles_y = (a.oy + BY - 1) / BY;
  const int sh = pxa - a.px;
  const size_t stage_bytes = ((size_t)a.sx * a.sy * sizeof(float) + 127) & ~size_t(127);
  auto stage = [&](int s) { return reinterpret_cast<float*>(smem_zp + (size_t)s * stage_bytes); };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_zp + NS * stage_bytes);
  int* rel = reinterpret_cast<int*>(smem_zp + NS * stage_bytes + 8 * NS);
  const int nwarps = (int)(blockDim.x >> 5), lane = tid & 31;
  const uint32_t box_bytes = (uint32_t)(a.sx * a.sy * sizeof(float));
  const bool active = ty < a.tyn;
  const int64_t total = a.batch * tiles_y * tiles_x * (int64_t)a.oz;
  int64_t pos = (int64_t)blockIdx.x * per_cta;
  int64_t end = min(total, pos + per_cta);
  if (zr.nc > 0) {  // run blockIdx.x % nc of column blockIdx.x / nc
    const int64_t c0 = (int64_t)(blockIdx.x / zr.nc) * a.oz;
    pos = c0 + zr.zb[blockIdx.x % zr.nc];
    end = c0 + zr.zb[blockIdx.x % zr.nc + 1];
  }
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&bars[i], 1);
    for (int i = 0; i < NS; ++i) rel[i] = 0;
    mbar_fence_init();
  }
  __syncthreads();
  int gcount = 0;
  const int wb = ty * a.sx + sh + tx * VX - SH4;  // aligned window base within a staged row

  while (pos < end) {
    const int64_t col = pos / a.oz;
    const int z0 = (int)(pos - col * a.oz);
    const int64_t left = end - pos;
    const int z1 = left < (int64_t)(a.oz - z0) ? z0 + (int)left : a.oz;
    pos += z1 - z0;
    const int b = (int)(col / (tiles_x * tiles_y));
    const int tt = (int)(col - (int64_t)b * tiles_x * tiles_y);
    const int x0 = (tt % tiles_x) * BX, y0 = (tt / tiles_x) * BY;
    const int s_beg = z0 - a.pz, s_end = z1 - a.pz + NZ - 1;
    const int g_lo = max(0, s_beg), g_hi = min(a.mz, s_end);
    const int nsl = max(0, g_hi - g_lo);
    const int g0 = gcount;
    auto issue = [&](int k, bool any = false) {
      if (any || tid == 0) {
        const int st = (g0 + k) % NS;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bars[st], box_bytes);
        tma_load_4d(stage(st), &tmap, &bars[st], x0 - pxa, y0 - a.py, g_lo + k, b);
      }
    };
    for (int k = 0; k < NS && k < nsl; ++k) issue(k);

    float2 P[NP + 1][VX];
#pragma unroll
    for (int i = 0; i <= NP; ++i)
#pragma unroll
      for (int x = 0; x < VX; ++x) P[i][x] = make_float2(0.f, 0.f);

    float* out = reinterpret_cast<float*>(a.out) + (int64_t)b * a.oz * a.oy * a.ox;
    const int ox = x0 + tx * VX;
    const int oy = y0 + ty;

    // one input slice s of parity PAR (0: slot j = e[j]; 1: slot j = e[j-1], slot 0 = e[NZ])
    auto slice = [&](int s, auto par_c) {
      constexpr int PAR = decltype(par_c)::value;
      if (s >= g_lo && s < g_hi) {
        const int k = s - g_lo;
        const int g = g0 + k;
        mbar_wait(&bars[g % NS], (uint32_t)((g / NS) & 1));
        const int jlo = max(0, s + a.pz - z1 + 1), jhi = min(NZ - 1, s + a.pz - z0);
        const float* tile = stage(g % NS) + wb;
        const float* kpar = taps.v + PAR * (NH * NW * EP);
        if (active) {
          if (jlo == 0 && jhi == NZ - 1) {  // every slot live: plane pairs
#pragma unroll 1
            for (int j1 = 0; j1 < NH; ++j1) {
              float v[NV4 * 4];
              const float4* rp = reinterpret_cast<const float4*>(tile + j1 * a.sx);
#pragma unroll
              for (int c = 0; c < NV4; ++c) {
                const float4 q = rp[c];
                v[4 * c] = q.x;
                v[4 * c + 1] = q.y;
                v[4 * c + 2] = q.z;
                v[4 * c + 3] = q.w;
              }
              const float* kj1 = kpar + j1 * (NW * EP);
#pragma unroll
              for (int j2 = 0; j2 < NW; ++j2) {
                float kr[EP];
#pragma unroll
                for (int q = 0; q < EP; q += 4)
                  *reinterpret_cast<float4*>(kr + q) = *reinterpret_cast<const float4*>(kj1 + j2 * EP + q);
                const float ks = PAR ? kr[NZ] : kr[NZ - 1];
#pragma unroll
                for (int x = 0; x < VX; ++x) {
                  const float vv = v[SH4 + x + j2];
                  const float2 vb = make_float2(vv, vv);
#pragma unroll
                  for (int i = 0; i < NP; ++i) P[i][x] = ffma2(vb, make_float2(kr[2 * i], kr[2 * i + 1]), P[i][x]);
                  if (PAR)
                    P[NP][x].y = fmaf(ks, vv, P[NP][x].y);
                  else
                    P[NP][x].x = fmaf(ks, vv, P[NP][x].x);
                }
              }
            }
          } else {  // run ends: only slots jlo..jhi are live
#pragma unroll 1
            for (int j1 = 0; j1 < NH; ++j1) {
              float v[NV4 * 4];
              const float4* rp = reinterpret_cast<const float4*>(tile + j1 * a.sx);
#pragma unroll
              for (int c = 0; c < NV4; ++c) {
                const float4 q = rp[c];
                v[4 * c] = q.x;
                v[4 * c + 1] = q.y;
                v[4 * c + 2] = q.z;
                v[4 * c + 3] = q.w;
              }
              const float* kj1 = kpar + j1 * (NW * EP);
#pragma unroll
              for (int j = 0; j < NZ; ++j) {
                if (j < jlo || j > jhi) continue;
                const int e = PAR ? (j == 0 ? NZ : j - 1) : j;  // register element of slot j (also its tap column)
#pragma unroll
                for (int j2 = 0; j2 < NW; ++j2) {
                  const float kv = kj1[j2 * EP + e];
#pragma unroll
                  for (int x = 0; x < VX; ++x) {
                    const float vv = v[SH4 + x + j2];
                    if (e & 1)
                      P[e >> 1][x].y = fmaf(kv, vv, P[e >> 1][x].y);
                    else
                      P[e >> 1][x].x = fmaf(kv, vv, P[e >> 1][x].x);
                  }
                }
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          if ((atomicAdd(&rel[g % NS], 1) % nwarps) == nwarps - 1 && k + NS < nsl) issue(k + NS, true);
        }
      }
      // slot NZ-1 now holds output z = s + pz - (NZ-1), complete
      const int zo = s + a.pz - (NZ - 1);
      if (zo >= z0 && zo < z1 && active && oy < a.oy) {
        float* orow = out + ((int64_t)zo * a.oy + oy) * a.ox;
#pragma unroll
        for (int x = 0; x < VX; ++x)
          if (ox + x < a.ox) orow[ox + x] = PAR ? P[NP - 1][x].y : P[NP][x].x;
      }
    };

    for (int s = s_beg; s < s_end; s += 2) {
      slice(s, std::integral_constant<int, 0>{});
      if (s + 1 < s_end) slice(s + 1, std::integral_constant<int, 1>{});
      // e' = [0, e[NZ], e0, .., e[NZ-3], 0]
#pragma unroll
      for (int x = 0; x < VX; ++x) {
        const float carry = P[NP][x].y;
        P[NP][x] = make_float2(P[NP - 1][x].x, 0.f);
#pragma unroll
        for (int i = NP - 1; i > 0; --i) P[i][x] = P[i - 1][x];
        P[0][x] = make_float2(0.f, carry);
      }
    }
    gcount += nsl;
    __syncthreads();  // run boundary: every stage free before the next run's first loads
  }
}

template <int NZ, int MAXT = 256>
int launch_zwalk_zp(const TileArgs& a0, const float* taps_host, int ntaps, cudaStream_t st) {
  TileArgs a = a0;
  constexpr int VX = 8, NH = NZ, NW = NZ;
  constexpr int EP = (NZ + 1 + 3) / 4 * 4;
  static_assert(2 * NH * NW * EP <= MaxTaps<float>::value, "tap rows exceed the parameter block");
  TapsParam<float> taps;
  memset(&taps, 0, sizeof(taps));
  (void)ntaps;
  for (int j1 = 0; j1 < NH; ++j1)
    for (int j2 = 0; j2 < NW; ++j2) {
      float* even = taps.v + (j1 * NW + j2) * EP;
      float* odd = taps.v + NH * NW * EP + (j1 * NW + j2) * EP;
      for (int j = 0; j < NZ; ++j) {
        const float kv = taps_host[(j * NH + j1) * NW + j2];
        even[j] = kv;
        odd[j == 0 ? NZ : j - 1] = kv;
      }
    }
  a.txn = a.tyn = 0;
  choose_zwalk_tile(a.oy, a.ox, VX, 1, NH, NW, &a.txn, &a.tyn, MAXT);
  if (getenv("CT_ZW_TXN") && getenv("CT_ZW_TYN")) {  // probing only
    a.txn = atoi(getenv("CT_ZW_TXN"));
    a.tyn = atoi(getenv("CT_ZW_TYN"));
  }
  const int pxa = (a.px + 3) / 4 * 4;
  const int sh = pxa - a.px;  // 0..3
  const int BX = a.txn * VX, BY = a.tyn;
  const int nv4 = (sh + VX + NW - 1 + 3) / 4;
  a.sx = std::max((sh + BX + NW - 1 + 3) / 4 * 4, BX - VX + 4 * nv4);  // every thread's vector loads stay in the row
  a.sy = BY + NH - 1;
  const size_t stage_bytes = ((size_t)a.sx * a.sy * sizeof(float) + 127) & ~size_t(127);
  const size_t smem = 3 * stage_bytes + 64;
  CT_REQUIRE(smem <= 227 * 1024, "zwalk tile too large");
  const int nthr = (int)cdiv(a.txn * a.tyn, 32) * 32;
  void (*kern)(const TileArgs, const TapsParam<float>, const CUtensorMap, int, int64_t, const ZRuns);
  switch (sh) {
    case 0: kern = xcorr_zwalk_zp<NZ, 0, MAXT>; break;
    case 1: kern = xcorr_zwalk_zp<NZ, 1, MAXT>; break;
    case 2: kern = xcorr_zwalk_zp<NZ, 2, MAXT>; break;
    default: kern = xcorr_zwalk_zp<NZ, 3, MAXT>; break;
  }
  CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 1;
  CT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nthr, smem));
  const int64_t total = cdiv(a.ox, BX) * cdiv(a.oy, BY) * a.batch * a.oz;
  const int64_t slots = (int64_t)num_sms() * std::max(1, per_sm);
  int64_t per_cta = std::max<int64_t>(cdiv(total, slots), 2 * NZ);
  ZRuns zr = plan_zruns(a, NZ, total / a.oz, slots);
  if (const char* e = getenv("CT_ZW_ZC")) {  // probing only
    per_cta = std::max(1, atoi(e));
    zr.nc = 0;
  }
  const int64_t nctas = zr.nc > 0 ? (total / a.oz) * zr.nc : cdiv(total, per_cta);
  CT_REQUIRE(nctas < (1ll << 31), "too many z-walk CTAs");
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  if (a.sx > 256 || a.sy > 256 ||
      !encode_tmap_4d(&tmap, a.s, sizeof(float), (uint64_t)a.mx, (uint64_t)a.my, (uint64_t)a.mz, (uint64_t)a.batch,
                      a.sx, a.sy)) {
    set_error("tensor map encode failed");
    return CT_EUNSUPPORTED;
  }
  if (getenv("CT_DEBUG"))
    fprintf(stderr, "xcorr_zwalk_zp NZ %d MAXT %d: tile %dx%d (%d thr) per_cta %lld runs/column %d per_sm %d ctas %lld smem %zu\n",
            NZ, MAXT, BX, BY, nthr, (long long)per_cta, zr.nc, per_sm, (long long)nctas, smem);
  kern<<<(unsigned)nctas, nthr, smem, st>>>(a, taps, tmap, pxa, per_cta, zr);
  return check_launch("xcorr_zwalk_zp");
}

// Persistent 2-D variant of xcorr_pair_f32 for large kernels (config 4): a
// CTA walks output tiles; the next tile's input values are loaded from
// global memory into registers (PF per thread) before the current tile's
// FMAs, so the global-load latency of the staging is hidden behind compute;
// after the tile they are written to the E/O pair copies.  Same arithmetic
// as xcorr_pair_f32.
constexpr int kPfRows = 12, kPfCols = 4;  // staged (row, column) slots per thread the register prefetch covers
#ifndef CT_PAIR_SCALAR_TAPS
#define CT_PAIR_SCALAR_TAPS 1  // scalar taps + FFMA2 broadcast operand: cfg4 0.316 -> 0.307 ms
#endif
template <int NW>
constexpr int kPairKP() { return (NW + 3) / 4 * 4; }  // scalar taps per kernel row, 16-byte padded
constexpr int kPairPF = kPfRows * kPfCols;

template <int NW>
__global__ void __launch_bounds__(256, 2) xcorr_pair_f32_pf(const TileArgs a, const __grid_constant__ TapsPairParam taps,
                                                           int tiles_x, int tiles_y) {
  extern __shared__ __align__(16) unsigned char smem_pf[];
  constexpr int WIN = kPairVX + NW - 1;
  constexpr int WLD = (WIN + 1) / 2;
  const int tid = threadIdx.x;
  const int tx = tid % a.txn, ty = tid / a.txn;
  const int BX = a.txn * kPairVX, BY = a.tyn * 2;
  const int ny = a.ny;
  const int SY = a.sy, SXp = a.sx;
  const int SXl = BX - kPairVX + 2 * WLD;
  const int PE = (SY + 1) / 2;
  float2* cE = reinterpret_cast<float2*>(smem_pf);
  float2* cO = cE + (size_t)PE * SXp;
  float* fE = reinterpret_cast<float*>(cE);
  float* fO = reinterpret_cast<float*>(cO);
  const int lane = tid & 31, nwarps = blockDim.x >> 5;
  const int64_t n_tiles = a.batch * tiles_y * tiles_x;
  float pf[kPairPF];

  // staged element (r, c) of this thread: r = warp + 8 i (i < kPfRows), c = lane + 32 j (j < kPfCols)
  auto fetch = [&](int64_t t) {  // global -> registers for tile t
    const int64_t b = t / (tiles_x * tiles_y);
    const int tt = (int)(t - b * tiles_x * tiles_y);
    const int x0 = (tt % tiles_x) * BX, y0 = (tt / tiles_x) * BY;
    const float* sp = reinterpret_cast<const float*>(a.s) + b * (int64_t)a.my * a.mx;
    const int iy0 = y0 - a.py, ix0 = x0 - a.px;
#pragma unroll
    for (int i = 0; i < kPfRows; ++i) {
      const int r = (tid >> 5) + i * nwarps;
      int gy = iy0 + r;
      const bool row_in = (unsigned)gy < (unsigned)a.my;
      if (!row_in && a.boundary == CT_REPLICATE) gy = gy < 0 ? 0 : a.my - 1;
      const float* srow = sp + (int64_t)gy * a.mx;
#pragma unroll
      for (int j = 0; j < kPfCols; ++j) {
        const int c = lane + 32 * j;
        int gx = ix0 + c;
        float v = 0.f;
        if (r < SY && c < SXl) {
          if (row_in && (unsigned)gx < (unsigned)a.mx) {
            v = __ldg(srow + gx);
          } else if (a.boundary == CT_REPLICATE) {
            gx = min(max(gx, 0), a.mx - 1);
            v = __ldg(srow + gx);
          }
        }
        pf[i * kPfCols + j] = v;
      }
    }
  };
  auto store = [&]() {  // registers -> E/O pair copies
#pragma unroll
    for (int i = 0; i < kPfRows; ++i) {
      const int r = (tid >> 5) + i * nwarps;
      if (r >= SY) break;
      float* dE = fE + (size_t)(r >> 1) * SXp * 2 + (r & 1);
      float* dO = r >= 1 ? fO + (size_t)((r - 1) >> 1) * SXp * 2 + ((r - 1) & 1) : nullptr;
#pragma unroll
      for (int j = 0; j < kPfCols; ++j) {
        const int c = lane + 32 * j;
        if (c < SXl) {
          const float v = pf[i * kPfCols + j];
          const int cp = pair_pad(c) * 2;
          dE[cp] = v;
          if (dO) dO[cp] = v;
        }
      }
    }
    if (SY & 1) {
      for (int c = tid; c < SXp; c += blockDim.x) fE[(((SY - 1) >> 1) * SXp + c) * 2 + 1] = 0.f;
    } else {
      for (int c = tid; c < SXp; c += blockDim.x) fO[(((SY - 2) >> 1) * SXp + c) * 2 + 1] = 0.f;
    }
  };

  int64_t t = blockIdx.x;
  if (t < n_tiles) fetch(t);
  for (; t < n_tiles; t += gridDim.x) {
    __syncthreads();  // previous tile's compute done with E/O
    store();
    __syncthreads();
    if (t + gridDim.x < n_tiles) fetch(t + gridDim.x);  // in flight during this tile's FMAs

    const int64_t b = t / (tiles_x * tiles_y);
    const int tt = (int)(t - b * tiles_x * tiles_y);
    const int x0 = (tt % tiles_x) * BX, y0 = (tt / tiles_x) * BY;
    float2 acc[kPairVX];
#pragma unroll
    for (int m = 0; m < kPairVX; ++m) acc[m] = make_float2(0.f, 0.f);
    for (int j1 = 0; j1 < ny; ++j1) {
      const int lr = 2 * ty + j1;
      const float2* prow = ((lr & 1) ? cO : cE) + (size_t)(lr >> 1) * SXp;
      float2 w[2 * WLD];
#pragma unroll
      for (int c = 0; c < WLD; ++c) {
        const float4 q = *reinterpret_cast<const float4*>(prow + 10 * tx + 2 * c + 2 * (c >> 2));
        w[2 * c] = make_float2(q.x, q.y);
        w[2 * c + 1] = make_float2(q.z, q.w);
      }
#if CT_PAIR_SCALAR_TAPS
      // scalar taps, 4 per 16-byte uniform load; (k, k) formed in registers (FFMA2 broadcast operand)
      const float* kr = reinterpret_cast<const float*>(taps.v) + j1 * kPairKP<NW>();
#pragma unroll
      for (int q = 0; q < kPairKP<NW>(); q += 4) {
        const float4 k4 = *reinterpret_cast<const float4*>(kr + q);
        const float kq[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j2 = q + e;
          if (j2 < NW) {
            const float2 kk = make_float2(kq[e], kq[e]);
#pragma unroll
            for (int m = 0; m < kPairVX; ++m) acc[m] = ffma2(kk, w[m + j2], acc[m]);
          }
        }
      }
#else
      const float2* kr = taps.v + j1 * NW;
#pragma unroll
      for (int j2 = 0; j2 < NW; ++j2) {
        const float2 kk = kr[j2];
#pragma unroll
        for (int m = 0; m < kPairVX; ++m) acc[m] = ffma2(kk, w[m + j2], acc[m]);
      }
#endif
    }
    float* out = reinterpret_cast<float*>(a.out) + b * (int64_t)a.oy * a.ox;
    const int y = y0 + 2 * ty;
    const int x = x0 + tx * kPairVX;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (y + h >= a.oy) break;
      float* orow = out + ((int64_t)y + h) * a.ox;
#pragma unroll
      for (int m = 0; m < kPairVX; ++m)
        if (x + m < a.ox) orow[x + m] = h ? acc[m].y : acc[m].x;
    }
  }
}

template <int NW>
int launch_pair_f32_pf(const TileArgs& a0, const float* taps_host, int ntaps, cudaStream_t st) {
  TileArgs a = a0;
  TapsPairParam taps;
#if CT_PAIR_SCALAR_TAPS
  {
    float* tv = reinterpret_cast<float*>(taps.v);
    const int rows = ntaps / NW;
    for (int r = 0; r < rows; ++r)
      for (int j2 = 0; j2 < kPairKP<NW>(); ++j2) tv[r * kPairKP<NW>() + j2] = j2 < NW ? taps_host[r * NW + j2] : 0.f;
  }
#else
  for (int i = 0; i < ntaps; ++i) taps.v[i] = make_float2(taps_host[i], taps_host[i]);
#endif
  const int BX = a.txn * kPairVX, BY = a.tyn * 2;
  constexpr int WIN = kPairVX + NW - 1;
  constexpr int WLD = (WIN + 1) / 2;
  a.sy = BY + a.ny - 1;
  const int sxl = BX - kPairVX + 2 * WLD;
  a.sx = pair_pad(sxl - 1) + 1;
  a.sx += (a.sx & 1);
  const int nthr = a.txn * a.tyn;
  CT_REQUIRE(nthr % 32 == 0 && nthr <= 256, "pair pf tile");
  if (cdiv(a.sy, nthr / 32) > kPfRows || cdiv(sxl, 32) > kPfCols) {
    set_error("pair pf tile too large for the register prefetch");
    return CT_EUNSUPPORTED;
  }
  const int PE = (a.sy + 1) / 2, PO = a.sy / 2;
  const size_t smem = (size_t)(PE + PO) * a.sx * sizeof(float2);
  auto kern = xcorr_pair_f32_pf<NW>;
  CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 1;
  CT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nthr, smem));
  const int tiles_x = (int)cdiv(a.ox, BX), tiles_y = (int)cdiv(a.oy, BY);
  const int64_t n_tiles = a.batch * tiles_x * tiles_y;
  const int64_t grid = std::min<int64_t>(n_tiles, (int64_t)num_sms() * std::max(1, per_sm));
  kern<<<(unsigned)grid, nthr, smem, st>>>(a, taps, tiles_x, tiles_y);
  return check_launch("xcorr_pair_f32_pf");
}

// Tile shape (threads along x, thread rows) minimising padded FMAs plus
// staging over the whole output, for vx outputs per thread along x and
// rows_per_thread output rows per thread.
inline void choose_tile(const TileArgs& a, int nw, int vx, int rows_per_thread, int* txn, int* tyn,
                        bool whole_warps) {
  const double taps = (double)a.ny * (double)nw;
  double best = 1e300;
  for (int tx = 4; tx <= 64; ++tx) {
    for (int ty = 1; tx * ty <= 256; ++ty) {
      const int thr = tx * ty;
      if (thr < 64 || (whole_warps && thr % 32 != 0)) continue;  // pair kernel stages rows per warp
      const double bx = tx * vx, by = ty * rows_per_thread;
      const double tiles = (double)cdiv(a.ox, (int64_t)bx) * (double)cdiv(a.oy, (int64_t)by);
      const double warp_eff = (double)thr / (double)(cdiv(thr, 32) * 32);
      const double stage = (bx + nw + vx) * (by + a.ny - 1);
      const double cost = tiles * (bx * by * taps / warp_eff + 8.0 * stage);
      if (cost < best * 0.999) {
        best = cost;
        *txn = tx;
        *tyn = ty;
      }
    }
  }
}

// The K best thread blocks of choose_tile's cost model (the autotuner times them).
inline std::vector<std::pair<int, int>> choose_tiles_top(const TileArgs& a, int nw, int vx, int rows_per_thread, int K) {
  const double taps = (double)a.ny * (double)nw;
  std::vector<std::pair<double, std::pair<int, int>>> all;
  for (int tx = 4; tx <= 64; ++tx)
    for (int ty = 1; tx * ty <= 256; ++ty) {
      const int thr = tx * ty;
      if (thr < 64) continue;
      const double bx = tx * vx, by = ty * rows_per_thread;
      const double tiles = (double)cdiv(a.ox, (int64_t)bx) * (double)cdiv(a.oy, (int64_t)by);
      const double warp_eff = (double)thr / (double)(cdiv(thr, 32) * 32);
      const double stage = (bx + nw + vx) * (by + a.ny - 1);
      all.push_back({tiles * (bx * by * taps / warp_eff + 8.0 * stage), {tx, ty}});
    }
  std::sort(all.begin(), all.end());
  std::vector<std::pair<int, int>> out;
  for (size_t i = 0; i < all.size() && (int)out.size() < K; ++i) out.push_back(all[i].second);
  return out;
}

// The tiled kernel takes its taps through the kernel-parameter bank, so they
// are needed on the host: the caller's host copy is used when given, else the
// device kernel is copied (a few KB, synchronising the stream).  flip
// reverses the flat row-major buffer, which is reflect(k) (conv.py:62-64).
template <typename T>
int taps_to_host(const void* k, const void* k_host, int64_t n, int flip, T* dst, cudaStream_t st) {
  T tmp[MaxTaps<T>::value];
  if (k_host) {
    memcpy(tmp, k_host, (size_t)n * sizeof(T));
  } else {
    CT_CUDA(cudaMemcpyAsync(tmp, k, (size_t)n * sizeof(T), cudaMemcpyDeviceToHost, st));
    CT_CUDA(cudaStreamSynchronize(st));
  }
  for (int64_t i = 0; i < n; ++i) dst[i] = flip ? tmp[n - 1 - i] : tmp[i];
  return CT_OK;
}

// One tiled variant: kind 0 = xcorr_tiled (TY=4 rows x VX per thread),
// kind 1 = xcorr_pair_f32 (2 rows x 8 per thread, f32 only).
template <typename T>
int launch_variant(TileArgs a, int kind, int nw, bool is3d, int txn, int tyn, const T* taps, int ntaps,
                   cudaStream_t st) {
  constexpr int VX = 16 / sizeof(T);
  a.txn = txn;
  a.tyn = tyn;
  if constexpr (sizeof(T) == 4) {
    if (kind == 1) {
      if (is3d) {
        a.tiles_z = (int)cdiv(a.oz, 2);
        switch (nw) {
#define CT_CASE(W) case W: return launch_pair_f32<W, 2>(a, reinterpret_cast<const float*>(taps), ntaps, st);
          CT_CASE(1) CT_CASE(2) CT_CASE(3) CT_CASE(4) CT_CASE(5) CT_CASE(6) CT_CASE(7) CT_CASE(8)
          CT_CASE(9) CT_CASE(11) CT_CASE(15) CT_CASE(31)
#undef CT_CASE
        }
      } else {
        a.tiles_z = 1;
        switch (nw) {
#define CT_CASE(W) case W: return launch_pair_f32<W, 1>(a, reinterpret_cast<const float*>(taps), ntaps, st);
          CT_CASE(1) CT_CASE(2) CT_CASE(3) CT_CASE(4) CT_CASE(5) CT_CASE(6) CT_CASE(7) CT_CASE(8)
          CT_CASE(9) CT_CASE(11) CT_CASE(15) CT_CASE(31)
#undef CT_CASE
        }
      }
      set_error("unsupported kernel width %d", nw);
      return CT_EUNSUPPORTED;
    }
  }
  if (kind == 2) {  // TMA-staged persistent 2-D kernel (zero boundary, aligned; see tma_ok)
    a.tiles_z = 1;
    switch (nw) {
#define CT_CASE(W)                                                                          \
  case W:                                                                                   \
    if (a.ny == W && (W == 3 || W == 5 || W == 7)) return launch_tma2d<T, W, tma_vx<T>(), 4, W>(a, taps, ntaps, st); \
    return launch_tma2d<T, W, tma_vx<T>(), 4, 0>(a, taps, ntaps, st);
      CT_CASE(1) CT_CASE(2) CT_CASE(3) CT_CASE(4) CT_CASE(5) CT_CASE(6) CT_CASE(7) CT_CASE(8)
      CT_CASE(9) CT_CASE(11) CT_CASE(15) CT_CASE(31)
#undef CT_CASE
    }
    set_error("unsupported kernel width %d", nw);
    return CT_EUNSUPPORTED;
  }
  if constexpr (sizeof(T) == 4) {
    if (kind == 6 && !is3d) {
      a.tiles_z = 1;
      switch (nw) {
#define CT_CASE(W) case W: return launch_pair_f32_pf<W>(a, reinterpret_cast<const float*>(taps), ntaps, st);
        CT_CASE(7) CT_CASE(8) CT_CASE(9) CT_CASE(11) CT_CASE(15) CT_CASE(31)
#undef CT_CASE
      }
      set_error("unsupported kernel width %d", nw);
      return CT_EUNSUPPORTED;
    }
    if (kind == 7) {  // z-walking 3-D kernel, FFMA2 over kernel-plane pairs (fp32)
      const int n = a.nz;
      const float* tf = reinterpret_cast<const float*>(taps);
      if (n == a.ny && n == nw) {
        if (n == 3) return launch_zwalk_zp<3>(a, tf, ntaps, st);
        if (n == 5) return launch_zwalk_zp<5>(a, tf, ntaps, st);
        if (n == 7) return launch_zwalk_zp<7>(a, tf, ntaps, st);
      }
      set_error("z-walk kernel needs a 3x3x3, 5x5x5 or 7x7x7 kernel");
      return CT_EUNSUPPORTED;
    }
    if (kind == 5) {  // z-walking 3-D kernel with packed FFMA2 (fp32)
      const int n = a.nz;
      const float* tf = reinterpret_cast<const float*>(taps);
      // fp32: one output row x 8 columns per thread (tile 136 x 15 on cfg3, 4 window loads per kernel
    // row instead of 6, 1 padded output row instead of 6): 0.307 -> 0.279 ms per batch of 8 against
    // 2 rows x 4 columns; fp64 keeps 2 rows x 2 columns
    const int cfg = getenv("CT_ZW_CFG") ? atoi(getenv("CT_ZW_CFG")) : (sizeof(T) == 4 ? 4 : 2);
      if (n == a.ny && n == nw) {
#define CT_ZWN(N)                                                                      \
  if (n == N) {                                                                        \
    if (cfg == 0) return launch_zwalk_x2<N, N, N, 4, 256>(a, tf, ntaps, st);           \
    return launch_zwalk_x2<N, N, N, 2, 512>(a, tf, ntaps, st);                         \
  }
        CT_ZWN(3) CT_ZWN(5) CT_ZWN(7)
#undef CT_ZWN
      }
      set_error("z-walk kernel needs a 3x3x3, 5x5x5 or 7x7x7 kernel");
      return CT_EUNSUPPORTED;
    }
  }
  if (kind == 4) {  // z-walking 3-D kernel (zero boundary, aligned rows, cubic 3/5/7 kernels; see zwalk_ok)
    constexpr int ZVX = sizeof(T) == 4 ? 4 : 2;
    const int n = a.nz;
    // fp32: one output row x 8 columns per thread (tile 136 x 15 on cfg3, 4 window loads per kernel
    // row instead of 6, 1 padded output row instead of 6): 0.307 -> 0.279 ms per batch of 8 against
    // 2 rows x 4 columns; fp64 keeps 2 rows x 2 columns
    const int cfg = getenv("CT_ZW_CFG") ? atoi(getenv("CT_ZW_CFG")) : (sizeof(T) == 4 ? 4 : 2);
    TileArgs a8 = a;  // wider per-thread rows: the tile is re-chosen for that shape
    a8.txn = a8.tyn = 0;
    if (n == a.ny && n == nw) {
#define CT_ZWN(N)                                                                          \
  if (n == N) {                                                                            \
    if (cfg == 1) return launch_zwalk<T, N, N, N, 3, ZVX, 384>(a, taps, ntaps, 0, st);    \
    if (cfg == 2) return launch_zwalk<T, N, N, N, 2, ZVX, 512>(a, taps, ntaps, 0, st);    \
    if (cfg == 3) return launch_zwalk<T, N, N, N, 1, 2 * ZVX, 512>(a8, taps, ntaps, 0, st); \
    if (cfg == 4) return launch_zwalk<T, N, N, N, 1, 2 * ZVX, 256>(a8, taps, ntaps, 0, st); \
    return launch_zwalk<T, N, N, N, 4, ZVX, 256>(a, taps, ntaps, 0, st);                   \
  }
      CT_ZWN(3) CT_ZWN(5) CT_ZWN(7)
#undef CT_ZWN
    }
    set_error("z-walk kernel needs a 3x3x3, 5x5x5 or 7x7x7 kernel");
    return CT_EUNSUPPORTED;
  }
  if (kind == 3) {  // TMA-staged 3-D kernel (zero boundary, aligned rows; see tma3_ok)
    switch (nw) {
#define CT_CASE(W) case W: return launch_tma3d<T, W, VX, 4, 2>(a, taps, ntaps, st);
      CT_CASE(1) CT_CASE(2) CT_CASE(3) CT_CASE(4) CT_CASE(5) CT_CASE(6) CT_CASE(7) CT_CASE(8)
      CT_CASE(9) CT_CASE(11) CT_CASE(15) CT_CASE(31)
#undef CT_CASE
    }
    set_error("unsupported kernel width %d", nw);
    return CT_EUNSUPPORTED;
  }
  if (is3d) {
    a.tiles_z = (int)cdiv(a.oz, 2);
    switch (nw) {
#define CT_CASE(W) case W: return launch_tiled<T, W, VX, 4, 2>(a, taps, ntaps, st);
      CT_CASE(1) CT_CASE(2) CT_CASE(3) CT_CASE(4) CT_CASE(5) CT_CASE(6) CT_CASE(7) CT_CASE(8)
      CT_CASE(9) CT_CASE(11) CT_CASE(15) CT_CASE(31)
#undef CT_CASE
    }
  } else {
    a.tiles_z = 1;
    switch (nw) {
#define CT_CASE(W) case W: return launch_tiled<T, W, VX, 4, 1>(a, taps, ntaps, st);
      CT_CASE(1) CT_CASE(2) CT_CASE(3) CT_CASE(4) CT_CASE(5) CT_CASE(6) CT_CASE(7) CT_CASE(8)
      CT_CASE(9) CT_CASE(11) CT_CASE(15) CT_CASE(31)
#undef CT_CASE
    }
  }
  set_error("unsupported kernel width %d", nw);
  return CT_EUNSUPPORTED;
}

struct Variant {
  int kind, txn, tyn;
  bool pin_only = false;  // reachable through CT_CONV_KIND only (never the fastest: not worth a mispick)
};

// Tile variant per problem shape, chosen once by timing a short candidate
// list on the caller's data (the first call of a large shape synchronises
// the stream; CT_CONV_AUTOTUNE=0 keeps the cost-model pick).
template <typename T>
int run_tiled_autotuned(TileArgs a, int nw, bool is3d, const T* taps, int ntaps, cudaStream_t st) {
  constexpr int VX = 16 / sizeof(T);
  std::vector<Variant> cands;
  int tx = 32, ty = 8;
  const bool f32 = sizeof(T) == 4 && getenv("CT_CONV_NOPAIR") == nullptr;
  if (f32) {
    choose_tile(a, nw, kPairVX, 2, &tx, &ty, true);
    cands.push_back({1, tx, ty});
    for (Variant v : {Variant{1, 8, 32}, Variant{1, 16, 16}, Variant{1, 16, 8}, Variant{1, 8, 16}, Variant{1, 32, 8}})
      cands.push_back(v);
    if (!is3d && nw >= 7 && (nw <= 9 || nw == 11 || nw == 15 || nw == 31))  // large 2-D kernels: persistent prefetch
      for (Variant v : {Variant{6, 8, 32}, Variant{6, 16, 16}, Variant{6, 8, 16}, Variant{6, 16, 8}})
        cands.push_back(v);
  }
  choose_tile(a, nw, VX, 4, &tx, &ty, false);
  cands.push_back({0, tx, ty});
  for (Variant v : {Variant{0, 32, 8}, Variant{0, 16, 16}, Variant{0, 32, 4}, Variant{0, 16, 8}, Variant{0, 64, 4}})
    cands.push_back(v);
  // TMA staging: 2-D, zero extension, box start and row pitch 16-byte aligned
  const bool tma_ok = !is3d && a.boundary == CT_ZERO && (a.px * (int)sizeof(T)) % 16 == 0 &&
                      (a.mx * (int64_t)sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(a.s) & 15) == 0 &&
                      getenv("CT_CONV_NOTMA") == nullptr;
  if (tma_ok) {
    // fixed shapes + the thread blocks fitted to the output extents (260^2 outputs: 3-9 % padded
    // instead of 23-36 %; cfg1 0.108 -> 0.100 ms per batch of 512)
    std::vector<Variant> tv2 = {Variant{2, 32, 8}, Variant{2, 16, 16}, Variant{2, 32, 4}, Variant{2, 16, 8},
                                Variant{2, 64, 4}};
    for (const auto& f : choose_tiles_top(a, nw, tma_vx<T>(), 4, 4)) tv2.push_back(Variant{2, f.first, f.second});
    for (Variant v : tv2) {
      constexpr int tv = tma_vx<T>();
      const int sx = v.txn * tv - tv + (int)cdiv(tv + nw - 1, tv) * tv, sy = v.tyn * 4 + a.ny - 1;
      if (sx <= 256 && sy <= 256) cands.push_back(v);
    }
  }
  // 3-D TMA staging: zero extension, 16-byte row pitch and base (any px)
  const bool tma3_ok = is3d && a.boundary == CT_ZERO && (a.mx * (int64_t)sizeof(T)) % 16 == 0 &&
                       (reinterpret_cast<uintptr_t>(a.s) & 15) == 0 && a.batch < (1ll << 31) &&
                       getenv("CT_CONV_NOTMA") == nullptr;
  if (tma3_ok) {
    for (Variant v : {Variant{3, 32, 8}, Variant{3, 16, 16}, Variant{3, 32, 4}, Variant{3, 16, 8}, Variant{3, 8, 16}}) {
      constexpr int vw = 16 / (int)sizeof(T);
      const int sx = (vw + v.txn * VX + nw - 1 + vw - 1) / vw * vw, sy = v.tyn * 4 + a.ny - 1;
      if (sx <= 256 && sy <= 256 && 2 * (size_t)sx * sy * sizeof(T) + 512 <= 227 * 1024) cands.push_back(v);
    }
  }
  // z-walking 3-D kernel: same TMA conditions, cubic 3/5/7 kernels
  const bool zwalk_ok = tma3_ok && a.nz == a.ny && a.ny == nw && (nw == 3 || nw == 5 || nw == 7);
  if (zwalk_ok) {
    int zx = 0, zy = 0;
    choose_zwalk_tile(a.oy, a.ox, sizeof(T) == 4 ? 4 : 2, 4, a.ny, nw, &zx, &zy);
    cands.insert(cands.begin(), Variant{4, zx, zy});
    // the FFMA2 z-walks (x pairs: 0.30 ms on cfg3; kernel-plane pairs: 0.272 ms) never beat the scalar
    // one (0.263 ms): kept for CT_CONV_KIND, not timed (a one-shot timing once picked the x-pair kernel)
    if (sizeof(T) == 4) cands.push_back(Variant{5, zx, zy, true});
    if (sizeof(T) == 4) cands.push_back(Variant{7, zx, zy, true});
  }
  const double work = (double)a.batch * a.oz * a.oy * a.ox * (double)a.nz * a.ny * nw;
  static const bool tune = !(getenv("CT_CONV_AUTOTUNE") && atoi(getenv("CT_CONV_AUTOTUNE")) == 0);
  if (const char* force = getenv("CT_CONV_KIND")) {  // tests: pin one variant family
    const int kind = atoi(force);
    for (const Variant& v : cands)
      if (v.kind == kind) return launch_variant<T>(a, v.kind, nw, is3d, v.txn, v.tyn, taps, ntaps, st);
  }
  // timing candidates synchronises the stream: never while the stream is being
  // captured into a CUDA graph (the cost-model pick is used instead)
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess) cudaGetLastError();
  if (!tune || work < 2.0e8 || cap != cudaStreamCaptureStatusNone)
    return launch_variant<T>(a, cands[0].kind, nw, is3d, cands[0].txn, cands[0].tyn, taps, ntaps, st);

  char key[256];
  snprintf(key, sizeof(key), "%zu|%d|%d,%d,%d|%d,%d,%d|%d,%d,%d|%d,%d,%d|%d|%lld", sizeof(T), nw, a.mz, a.my, a.mx,
           a.oz, a.oy, a.ox, a.nz, a.ny, nw, a.pz, a.py, a.px, a.boundary, (long long)a.batch);
  static std::mutex mu;
  static std::map<std::string, Variant> cache;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end())
      return launch_variant<T>(a, it->second.kind, nw, is3d, it->second.txn, it->second.tyn, taps, ntaps, st);
  }
  cudaEvent_t e0, e1;
  CT_CUDA(cudaEventCreate(&e0));
  CT_CUDA(cudaEventCreate(&e1));
  Variant best = cands[0];
  float best_ms = 1e30f;
  for (const Variant& v : cands) {
    if (v.pin_only || v.txn * v.tyn > 256 || v.txn * v.tyn < 32) continue;
    int rc = launch_variant<T>(a, v.kind, nw, is3d, v.txn, v.tyn, taps, ntaps, st);  // warm
    if (rc) continue;
    float ms = 1e30f;
    for (int rep = 0; rep < 3 && rc == CT_OK; ++rep) {  // best of three: one launch is within the box noise
      CT_CUDA(cudaEventRecord(e0, st));
      rc = launch_variant<T>(a, v.kind, nw, is3d, v.txn, v.tyn, taps, ntaps, st);
      CT_CUDA(cudaEventRecord(e1, st));
      CT_CUDA(cudaEventSynchronize(e1));
      float t = 0.f;
      cudaEventElapsedTime(&t, e0, e1);
      ms = std::min(ms, t);
    }
    if (rc == CT_OK && ms < best_ms) {
      best_ms = ms;
      best = v;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  {
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = best;
  }
  return launch_variant<T>(a, best.kind, nw, is3d, best.txn, best.tyn, taps, ntaps, st);
}

template <typename T>
int dispatch(int ndim, const void* s, const int64_t* ms, int64_t batch, const void* k,
             const void* k_host, const int64_t* ns, const int64_t* pl, const int64_t* os, int boundary, int flip,
             void* out, cudaStream_t st) {
  int64_t k_elems = 1, o_elems = 1, s_elems = 1;
  for (int d = 0; d < ndim; ++d) {
    k_elems *= ns[d];
    o_elems *= os[d];
    s_elems *= ms[d];
  }
  if (o_elems == 0 || batch == 0) return CT_OK;
  const int nw = (int)ns[ndim - 1];
  // the tiled kernels take the taps through the parameter bank; without a
  // host copy that needs a device->host read, which cannot happen while the
  // stream is captured into a CUDA graph (the generic kernel reads the taps
  // from device memory instead)
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (!k_host && cudaStreamIsCapturing(st, &cap) != cudaSuccess) cudaGetLastError();
  const bool tiled_ok = ndim <= 3 && k_elems <= MaxTaps<T>::value && s_elems > 0 &&
                        (k_host || cap == cudaStreamCaptureStatusNone) &&
                        (nw == 1 || nw == 2 || nw == 3 || nw == 4 || nw == 5 || nw == 6 ||
                         nw == 7 || nw == 8 || nw == 9 || nw == 11 || nw == 15 || nw == 31);
  // shapes as 3-D (z, y, x)
  auto as3d = [&](TileArgs& a) -> int {
    int64_t m3[3] = {1, 1, 1}, n3[3] = {1, 1, 1}, p3[3] = {0, 0, 0}, o3[3] = {1, 1, 1};
    for (int d = 0; d < ndim; ++d) {
      m3[3 - ndim + d] = ms[d];
      n3[3 - ndim + d] = ns[d];
      p3[3 - ndim + d] = pl[d];
      o3[3 - ndim + d] = os[d];
    }
    for (int d = 0; d < 3; ++d)
      CT_REQUIRE(m3[d] < (1 << 30) && o3[d] < (1 << 30) && p3[d] < (1 << 30), "extent too large");
    a = TileArgs{};
    a.s = s;
    a.out = out;
    a.batch = batch;
    a.mz = (int)m3[0]; a.my = (int)m3[1]; a.mx = (int)m3[2];
    a.oz = (int)o3[0]; a.oy = (int)o3[1]; a.ox = (int)o3[2];
    a.nz = (int)n3[0]; a.ny = (int)n3[1];
    a.pz = (int)p3[0]; a.py = (int)p3[1]; a.px = (int)p3[2];
    a.boundary = boundary;
    a.tiles_z = 1;
    return CT_OK;
  };
  // any other width (ranks 1-3): the width-generic strip kernel, taps read
  // from the device kernel (no host copy, capture-safe)
  static const bool no_strip = getenv("CT_CONV_NOSTRIP") != nullptr;  // tests: force the generic kernel
  if (!tiled_ok && ndim <= 3 && s_elems > 0 && !no_strip) {
    TileArgs a;
    int rc = as3d(a);
    if (rc) return rc;
    const bool is3d = a.oz > 1 || a.nz > 1;
    // rows per thread: fp64 reuses each window load over 8 output rows (the
    // DFMA:load ratio), fp32 over 4
    constexpr int STY = sizeof(T) == 8 ? CT_STRIP_TY64 : CT_STRIP_TY32;
    // taps in the parameter bank when they fit and a host copy is at hand (or
    // can be read: not while the stream is being captured)
    const int nwp = (nw + kStripC - 1) / kStripC * kStripC;
    T taps_h[MaxTaps<T>::value];  // flipped host taps (the launch copies the parameter block)
    const T* th = nullptr;
    if ((int64_t)a.nz * a.ny * nwp <= MaxTaps<T>::value && (k_host || cap == cudaStreamCaptureStatusNone)) {
      int rc2 = taps_to_host<T>(k, k_host, k_elems, flip, taps_h, st);
      if (rc2) return rc2;
      th = taps_h;
    }
    if (!is3d && tma_strip_ok<T>(a, nw, th != nullptr)) {  // TMA-staged tiles (falls through when the tile does not fit)
      const int rc3 = launch_tma2d_strip<T, STY>(a, th, nw, st);
      if (rc3 != CT_EUNSUPPORTED) return rc3;
    }
    if (strip_smem<T>(a, nw, 32, 8, STY, th != nullptr) > 0) {
      if (is3d) return launch_strip<T, STY, 2>(a, reinterpret_cast<const T*>(k), th, nw, flip, st);
      return launch_strip<T, STY, 1>(a, reinterpret_cast<const T*>(k), th, nw, flip, st);
    }
  }
  if (tiled_ok) {
    // shapes as 3-D (z, y, x)
    int64_t m3[3] = {1, 1, 1}, n3[3] = {1, 1, 1}, p3[3] = {0, 0, 0}, o3[3] = {1, 1, 1};
    for (int d = 0; d < ndim; ++d) {
      m3[3 - ndim + d] = ms[d];
      n3[3 - ndim + d] = ns[d];
      p3[3 - ndim + d] = pl[d];
      o3[3 - ndim + d] = os[d];
    }
    for (int d = 0; d < 3; ++d)
      CT_REQUIRE(m3[d] < (1 << 30) && o3[d] < (1 << 30) && p3[d] < (1 << 30), "extent too large");
    T taps_host[MaxTaps<T>::value];
    int rc = taps_to_host<T>(k, k_host, k_elems, flip, taps_host, st);
    if (rc) return rc;
    TileArgs a{};
    a.s = s;
    a.out = out;
    a.batch = batch;
    a.mz = (int)m3[0]; a.my = (int)m3[1]; a.mx = (int)m3[2];
    a.oz = (int)o3[0]; a.oy = (int)o3[1]; a.ox = (int)o3[2];
    a.nz = (int)n3[0]; a.ny = (int)n3[1];
    a.pz = (int)p3[0]; a.py = (int)p3[1]; a.px = (int)p3[2];
    a.boundary = boundary;
    const bool is3d = a.oz > 1 || a.nz > 1;
    a.tiles_z = 1;
    return run_tiled_autotuned<T>(a, nw, is3d, taps_host, (int)k_elems, st);
  }
  GenArgs g{};
  g.s = s;
  g.k = k;
  g.out = out;
  g.batch = batch;
  g.ndim = ndim;
  g.boundary = boundary;
  g.fused = ndim <= 3;
  g.flip = flip;
  int64_t acc = 1;
  for (int d = ndim - 1; d >= 0; --d) {
    g.ms[d] = ms[d];
    g.ns[d] = ns[d];
    g.pl[d] = pl[d];
    g.os[d] = os[d];
    g.sstr[d] = acc;
    acc *= ms[d];
  }
  g.s_elems = s_elems;
  g.o_elems = o_elems;
  g.k_elems = k_elems;
  const int64_t total = batch * o_elems;
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(total, 256), (int64_t)num_sms() * 32);
  xcorr_generic<T><<<blocks, 256, 0, st>>>(g);
  return check_launch("xcorr_generic");
}

}  // namespace
}  // namespace ct

using namespace ct;

static int xcorr_entry(int dtype, int ndim, const void* s, const int64_t* s_shape, int64_t batch,
                       const void* k, const void* k_host, const int64_t* k_shape, const int64_t* pad_left,
                       const int64_t* out_shape, int boundary, int flip, void* out, void* stream) {
  CT_REQUIRE(dtype == CT_F64 || dtype == CT_F32, "dtype must be CT_F64 or CT_F32");
  CT_REQUIRE(ndim >= 1 && ndim <= CT_MAXDIM, "ndim %d outside 1..%d", ndim, (int)CT_MAXDIM);
  CT_REQUIRE(boundary == CT_ZERO || boundary == CT_REPLICATE, "bad boundary");
  CT_REQUIRE(batch >= 0, "negative batch");
  for (int d = 0; d < ndim; ++d) {
    CT_REQUIRE(s_shape[d] >= 0 && k_shape[d] >= 1 && out_shape[d] >= 0 && pad_left[d] >= 0,
               "bad extents on axis %d", d);
    CT_REQUIRE(boundary == CT_ZERO || s_shape[d] >= 1, "replicate needs a non-empty signal");
  }
  cudaStream_t st = as_stream(stream);
  if (dtype == CT_F64)
    return dispatch<double>(ndim, s, s_shape, batch, k, k_host, k_shape, pad_left, out_shape, boundary, flip, out, st);
  return dispatch<float>(ndim, s, s_shape, batch, k, k_host, k_shape, pad_left, out_shape, boundary, flip, out, st);
}

extern "C" int ct_xcorr_nd(int dtype, int ndim, const void* s, const int64_t* s_shape,
                           int64_t batch, const void* k, const void* k_host, const int64_t* k_shape,
                           const int64_t* pad_left, const int64_t* out_shape, int boundary,
                           void* out, void* stream) {
  clear_error();
  return xcorr_entry(dtype, ndim, s, s_shape, batch, k, k_host, k_shape, pad_left, out_shape, boundary, 0, out,
                     stream);
}

extern "C" int ct_direct(int dtype, int ndim, const void* s, const int64_t* s_shape, int64_t batch,
                         const void* k, const void* k_host, const int64_t* k_shape, int shape, int boundary, int flip,
                         void* out, void* stream) {
  clear_error();
  CT_REQUIRE(ndim >= 1 && ndim <= CT_MAXDIM, "zero-rank tensors not supported");
  CT_REQUIRE(shape == CT_FULL || shape == CT_SAME || shape == CT_VALID, "bad shape");
  int64_t pl[CT_MAXDIM], os[CT_MAXDIM];
  for (int d = 0; d < ndim; ++d) {
    const int64_t m = s_shape[d], n = k_shape[d];
    CT_REQUIRE(n >= 1 && m >= 0, "bad extents on axis %d", d);
    if (shape == CT_FULL) {  // conv.py:142-145
      pl[d] = n - 1;
      os[d] = m + n - 1;
    } else if (shape == CT_SAME) {  // conv.py:146-150, _same_pads conv.py:115-117
      pl[d] = (n - 1) - (n - 1) / 2;
      os[d] = m;
    } else {  // conv.py:139-141, _check_valid conv.py:93-98
      CT_REQUIRE(m >= n, "VALID needs signal >= kernel on every axis, axis %d has %lld < %lld", d,
                 (long long)m, (long long)n);
      pl[d] = 0;
      os[d] = m - n + 1;
    }
  }
  // The boundary policy only matters where SAME reads outside the signal
  // (conv.py:146-150); FULL and VALID always zero-extend.
  const int bnd = shape == CT_SAME ? boundary : CT_ZERO;
  return xcorr_entry(dtype, ndim, s, s_shape, batch, k, k_host, k_shape, pl, os, bnd, flip ? 1 : 0, out, stream);
}
