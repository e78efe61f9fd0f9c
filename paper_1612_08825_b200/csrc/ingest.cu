// Frame ingestion (SURVEY.md 8(f) "next" row 4): PGM rasters travel to the
// device as their raw 8- or 16-bit samples (1-2 bytes per pixel instead of 8)
// and are decoded there exactly like tensor.image_read_pgm
// (/root/reference/pkg/src/convtact/tensor.py:104-136): float64(sample) /
// maxval, 16-bit samples big-endian.
#include <algorithm>

#include "common.cuh"

namespace ct {
namespace {

template <int BYTES>
__global__ void decode_kernel(const unsigned char* __restrict__ raw, int64_t n, double maxval, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned v;
    if (BYTES == 1) {
      v = raw[i];
    } else {
      v = ((unsigned)raw[2 * i] << 8) | (unsigned)raw[2 * i + 1];  // big-endian u16
    }
    out[i] = __ddiv_rn((double)v, maxval);
  }
}

}  // namespace
}  // namespace ct

using namespace ct;

extern "C" int ct_decode_samples(int bytes_per_sample, const void* raw, int64_t n, double maxval, double* out,
                                 void* stream) {
  clear_error();
  CT_REQUIRE(bytes_per_sample == 1 || bytes_per_sample == 2, "samples must be 1 or 2 bytes");
  CT_REQUIRE(n >= 0 && maxval > 0.0, "bad sample count or maxval");
  if (n == 0) return CT_OK;
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(n, 256), (int64_t)num_sms() * 32);
  cudaStream_t st = as_stream(stream);
  if (bytes_per_sample == 1)
    decode_kernel<1><<<blocks, 256, 0, st>>>((const unsigned char*)raw, n, maxval, out);
  else
    decode_kernel<2><<<blocks, 256, 0, st>>>((const unsigned char*)raw, n, maxval, out);
  return check_launch("decode_samples");
}
