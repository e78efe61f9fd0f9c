// Streaming probe shaped like ttc_moments_kernel: CTA = (band, video), walks
// F frames of its video; box = (BR+1) rows x 256 f64 at row (v*F + f)*H + band*BR.
// mode 0: wait frame f, consume, issue f+NB (plain ring)
// mode 1: pair ring: wait f and f+1 (f resident), issue f+NB after pair f
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include "../paper_1612_08825_b200/csrc/tma.cuh"
using namespace ct;

template <int NB>
__global__ void __launch_bounds__(256) probe(const __grid_constant__ CUtensorMap tm, int BR, int F, int H, int mode,
                                             double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const size_t bb = ((size_t)(BR + 1) * 256 * 8 + 8 * 8 + 127) & ~size_t(127);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + NB * bb);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NB; ++i) mbar_init(&bars[i], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int band = blockIdx.x;
  const int64_t v = blockIdx.z;
  const int64_t row0 = v * F * (int64_t)H + band * BR;
  auto issue = [&](int f) {
    if (threadIdx.x == 0) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&bars[f % NB], (uint32_t)((BR + 1) * 256 * 8));
      tma_load_2d(sm + (f % NB) * bb, &tm, &bars[f % NB], 0, (int)(row0 + (int64_t)f * H));
    }
  };
  for (int f = 0; f < NB && f < F; ++f) issue(f);
  double acc = 0;
  const int n = mode == 1 ? F - 1 : F;
  for (int i = 0; i < n; ++i) {
    mbar_wait(&bars[i % NB], (i / NB) & 1);
    if (mode == 1) mbar_wait(&bars[(i + 1) % NB], ((i + 1) / NB) & 1);
    acc += reinterpret_cast<const double*>(sm + (i % NB) * bb)[threadIdx.x];
    __syncthreads();
    if (i + NB < F) issue(i + NB);
  }
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  const int V = 256, F = 64, H = 256;
  const int64_t bytes = (int64_t)V * F * H * 256 * 8;
  double* d;
  cudaMalloc(&d, bytes);
  cudaMemset(d, 0, bytes);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  void* fnp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto fn = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  const int64_t rows = bytes / (256 * 8);
  for (int BR : {16, 32}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {256, (cuuint64_t)rows};
    cuuint64_t str[1] = {256 * 8};
    cuuint32_t box[2] = {256, (cuuint32_t)(BR + 1)};
    cuuint32_t es[2] = {1, 1};
    fn(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const size_t bb = ((size_t)(BR + 1) * 256 * 8 + 64 + 127) & ~size_t(127);
    for (int nb : {2, 3, 4, 6}) {
      const size_t smem = nb * bb + 64;
      if (smem > 227 * 1024) continue;
      auto kern = nb == 2 ? probe<2> : nb == 3 ? probe<3> : nb == 4 ? probe<4> : probe<6>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
      for (int mode : {0, 1}) {
        if (mode == 1 && nb < 3) continue;
        dim3 grid(H / BR, 1, V);
        kern<<<grid, 256, smem>>>(tm, BR, F, H, mode, out);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) kern<<<grid, 256, smem>>>(tm, BR, F, H, mode, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("BR %2d NB %d (%3.0f KB, %d CTA/SM) mode %d: %.3f ms  %.0f GB/s (frame bytes) %s\n", BR, nb,
               smem / 1024.0, per_sm, mode, ms / 3, 3.0 * bytes / (ms * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
