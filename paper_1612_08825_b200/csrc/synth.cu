// Synthetic approach frames on the device: synth.zoom_frame with the
// Catmull-Rom taps of synth._axis_taps (synth.py:88-126), evaluated op by op
// like numpy (rounded products and sums, no contraction) so float64 frames
// are bit-identical to the reference generator.  Used to produce benchmark
// and test inputs at sizes where the CPU generator is too slow.
#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace ct {
namespace {

struct Taps4 {
  int i[4];
  double w[4];
};

__device__ __forceinline__ Taps4 axis_taps(int p, int size, double center, double m) {
  // src = center + (p - center) / magnification
  const double src = __dadd_rn(center, __ddiv_rn(__dsub_rn((double)p, center), m));
  const double fl = floor(src);
  const int64_t i0 = (int64_t)fl;
  const double f = __dsub_rn(src, (double)i0);
  const double f2 = __dmul_rn(f, f);
  const double f3 = __dmul_rn(f2, f);
  Taps4 t;
  for (int b = 0; b < 4; ++b) {
    int64_t ii = i0 - 1 + b;
    ii = ii < 0 ? 0 : (ii > size - 1 ? size - 1 : ii);
    t.i[b] = (int)ii;
  }
  t.w[0] = __dsub_rn(__dadd_rn(__dmul_rn(-0.5, f3), f2), __dmul_rn(0.5, f));
  t.w[1] = __dadd_rn(__dsub_rn(__dmul_rn(1.5, f3), __dmul_rn(2.5, f2)), 1.0);
  t.w[2] = __dadd_rn(__dadd_rn(__dmul_rn(-1.5, f3), __dmul_rn(2.0, f2)), __dmul_rn(0.5, f));
  t.w[3] = __dsub_rn(__dmul_rn(0.5, f3), __dmul_rn(0.5, f2));
  return t;
}

constexpr int kMagsPerLaunch = 1024;
struct MagsParam {
  double m[kMagsPerLaunch];
};

template <typename T>
__global__ void zoom_kernel(const double* __restrict__ tex, int h, int w, double fx, double fy,
                            const __grid_constant__ MagsParam mags, int64_t n, T* __restrict__ out) {
  const int64_t per = (int64_t)h * w;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * per; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / per;
    const int64_t r = i - t * per;
    const int y = (int)(r / w), x = (int)(r - (int64_t)y * w);
    const double m = mags.m[t];
    double val;
    if (m == 1.0) {
      val = tex[r];
    } else {
      const Taps4 tx = axis_taps(x, w, fx, m);
      const Taps4 ty = axis_taps(y, h, fy, m);
      // tmp[iy][x] = sum_b wx_b * tex[iy][ix_b]; out = sum_a wy_a * tmp[iy_a][x]
      double acc = 0.0;
      for (int a = 0; a < 4; ++a) {
        const double* row = tex + (int64_t)ty.i[a] * w;
        double tmp = 0.0;
        for (int b = 0; b < 4; ++b) tmp = __dadd_rn(tmp, __dmul_rn(tx.w[b], row[tx.i[b]]));
        acc = __dadd_rn(acc, __dmul_rn(ty.w[a], tmp));
      }
      val = acc;
    }
    out[i] = (T)val;
  }
}

}  // namespace
}  // namespace ct

using namespace ct;

extern "C" size_t ct_zoom_frames_workspace_bytes(int64_t h, int64_t w) {
  (void)h;
  (void)w;
  return 0;
}

extern "C" int ct_zoom_frames(int dtype, const double* texture, int64_t h, int64_t w, double foe_x, double foe_y,
                              const double* mags_host, int64_t n, void* frames, void* workspace,
                              size_t workspace_bytes, void* stream) {
  (void)workspace;
  (void)workspace_bytes;
  clear_error();
  CT_REQUIRE(dtype == CT_F64 || dtype == CT_F32, "dtype must be CT_F64 or CT_F32");
  CT_REQUIRE(h >= 1 && w >= 1 && h < (1 << 30) && w < (1 << 30) && n >= 0, "bad extents");
  for (int64_t t = 0; t < n; ++t)
    CT_REQUIRE(mags_host[t] >= 1.0, "magnification must be >= 1, got %g", mags_host[t]);
  if (n == 0) return CT_OK;
  cudaStream_t st = as_stream(stream);
  // magnifications travel in the kernel-parameter bank, 1024 frames per launch
  const size_t esz = dtype == CT_F64 ? 8 : 4;
  for (int64_t t0 = 0; t0 < n; t0 += kMagsPerLaunch) {
    const int64_t cnt = std::min<int64_t>(kMagsPerLaunch, n - t0);
    MagsParam mp;
    for (int64_t t = 0; t < cnt; ++t) mp.m[t] = mags_host[t0 + t];
    const int64_t total = cnt * h * w;
    const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(total, 256), (int64_t)num_sms() * 32);
    char* dst = reinterpret_cast<char*>(frames) + (size_t)t0 * h * w * esz;
    if (dtype == CT_F64)
      zoom_kernel<double><<<blocks, 256, 0, st>>>(texture, (int)h, (int)w, foe_x, foe_y, mp, cnt, (double*)dst);
    else
      zoom_kernel<float><<<blocks, 256, 0, st>>>(texture, (int)h, (int)w, foe_x, foe_y, mp, cnt, (float*)dst);
    int rc = check_launch("zoom");
    if (rc) return rc;
  }
  return CT_OK;
}
