// Gradient fields (SURVEY.md 8(f) "next" row 3): kernels.gradient
// (/root/reference/pkg/src/convtact/kernels.py:63-72) fused into one pass.
// For each pixel: ex, ey = SAME/REPLICATE cross-correlations with the named
// pair (taps in row-major order with FMA, like the direct-conv loops, so ex/ey
// are bit-identical to the reference), then mag = hypot(ex, ey) and
// dir = atan2(ey, ex) in the epilogue -- one read of the image, four writes,
// no intermediate round trip.
#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace ct {
namespace {

constexpr int kMaxGradTaps = 64;

template <typename T>
struct GradTaps {
  T kx[kMaxGradTaps], ky[kMaxGradTaps];
};

template <typename T>
__device__ __forceinline__ T fma_t(T a, T b, T c);
template <>
__device__ __forceinline__ double fma_t(double a, double b, double c) {
  return fma(a, b, c);
}
template <>
__device__ __forceinline__ float fma_t(float a, float b, float c) {
  return fmaf(a, b, c);
}

template <typename T>
__global__ void __launch_bounds__(256) gradient_kernel(const T* __restrict__ img, int64_t n_images, int h, int w,
                                                       int kh, int kw, const __grid_constant__ GradTaps<T> taps,
                                                       T* ex, T* ey, T* mag, T* dir) {
  // SAME anchor: left pad ceil((n-1)/2) (conv.py:115-117), edge replicate
  const int py = (kh - 1) - (kh - 1) / 2, px = (kw - 1) - (kw - 1) / 2;
  const int64_t per = (int64_t)h * w;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_images * per;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / per;
    const int64_t r = i - b * per;
    const int y = (int)(r / w), x = (int)(r - (int64_t)y * w);
    const T* src = img + b * per;
    T sx = T(0), sy = T(0);
    for (int j0 = 0; j0 < kh; ++j0) {
      const int yy = min(max(y - py + j0, 0), h - 1);
      for (int j1 = 0; j1 < kw; ++j1) {
        const int xx = min(max(x - px + j1, 0), w - 1);
        const T v = src[(int64_t)yy * w + xx];
        sx = fma_t(taps.kx[j0 * kw + j1], v, sx);
        sy = fma_t(taps.ky[j0 * kw + j1], v, sy);
      }
    }
    ex[i] = sx;
    ey[i] = sy;
    mag[i] = hypot(sx, sy);
    dir[i] = atan2(sy, sx);
  }
}

}  // namespace
}  // namespace ct

using namespace ct;

extern "C" int ct_gradient(int dtype, const void* img, int64_t n_images, int64_t h, int64_t w, const double* kx_host,
                           const double* ky_host, int64_t kh, int64_t kw, void* ex, void* ey, void* mag, void* dir,
                           void* stream) {
  clear_error();
  CT_REQUIRE(dtype == CT_F64 || dtype == CT_F32, "dtype must be CT_F64 or CT_F32");
  CT_REQUIRE(h >= 1 && w >= 1 && h < (1 << 30) && w < (1 << 30) && n_images >= 0, "bad image extents");
  CT_REQUIRE(kh >= 1 && kw >= 1 && kh * kw <= kMaxGradTaps, "kernel pair must have 1..%d taps", kMaxGradTaps);
  const int64_t total = n_images * h * w;
  if (total == 0) return CT_OK;
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(total, 256), (int64_t)num_sms() * 32);
  cudaStream_t st = as_stream(stream);
  if (dtype == CT_F64) {
    GradTaps<double> t;
    for (int i = 0; i < kh * kw; ++i) {
      t.kx[i] = kx_host[i];
      t.ky[i] = ky_host[i];
    }
    gradient_kernel<double><<<blocks, 256, 0, st>>>((const double*)img, n_images, (int)h, (int)w, (int)kh, (int)kw, t,
                                                    (double*)ex, (double*)ey, (double*)mag, (double*)dir);
  } else {
    GradTaps<float> t;
    for (int i = 0; i < kh * kw; ++i) {
      t.kx[i] = (float)kx_host[i];
      t.ky[i] = (float)ky_host[i];
    }
    gradient_kernel<float><<<blocks, 256, 0, st>>>((const float*)img, n_images, (int)h, (int)w, (int)kh, (int)kw, t,
                                                   (float*)ex, (float*)ey, (float*)mag, (float*)dir);
  }
  return check_launch("gradient");
}
