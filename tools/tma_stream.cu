// Read-only HBM streaming probe: plain LDG.128 vs TMA 2-D boxes (rows x 256 f64)
// through an NB-deep mbarrier ring, to find what the moments kernel's data
// pipeline can reach.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I../include tools/tma_stream.cu -o /tmp/tma_stream -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include "../paper_1612_08825_b200/csrc/tma.cuh"
using namespace ct;

__global__ void ldg_sum(const double4* __restrict__ p, int64_t n, double* out) {
  double acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double4 v = p[i];
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1.2345) out[0] = acc;
}

template <int NB>
__global__ void tma_sum(const __grid_constant__ CUtensorMap tm, int rows_box, int64_t total_rows, int boxes_per_cta,
                        double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const size_t bb = (size_t)rows_box * 256 * 8;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + NB * bb);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NB; ++i) mbar_init(&bars[i], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t first = (int64_t)blockIdx.x * boxes_per_cta;
  auto issue = [&](int k) {
    if (threadIdx.x == 0) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&bars[k % NB], (uint32_t)bb);
      tma_load_2d(sm + (k % NB) * bb, &tm, &bars[k % NB], 0, (int)((first + k) * rows_box));
    }
  };
  for (int k = 0; k < NB && k < boxes_per_cta; ++k) issue(k);
  double acc = 0;
  for (int k = 0; k < boxes_per_cta; ++k) {
    mbar_wait(&bars[k % NB], (k / NB) & 1);
    const double* b = reinterpret_cast<const double*>(sm + (k % NB) * bb);
    acc += b[threadIdx.x];
    __syncthreads();
    if (k + NB < boxes_per_cta) issue(k + NB);
  }
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  const int64_t bytes = 8ll << 30;
  double* d;
  cudaMalloc(&d, bytes);
  cudaMemset(d, 0, bytes);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int g : {sms * 4, sms * 8, sms * 16}) {
    ldg_sum<<<g, 512>>>((const double4*)d, bytes / 32, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) ldg_sum<<<g, 512>>>((const double4*)d, bytes / 32, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("ldg grid %d: %.0f GB/s\n", g, 5.0 * bytes / (ms * 1e-3) / 1e9);
  }
  void* fnp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto fn = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  const int64_t rows = bytes / (256 * 8);
  for (int rb : {8, 16, 17, 32, 64}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {256, (cuuint64_t)rows};
    cuuint64_t str[1] = {256 * 8};
    cuuint32_t box[2] = {256, (cuuint32_t)rb};
    cuuint32_t es[2] = {1, 1};
    fn(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const size_t bb = (size_t)rb * 256 * 8;
    for (int nb : {2, 3, 4, 6}) {
      const size_t smem = nb * bb + 64;
      if (smem > 227 * 1024) continue;
      auto kern = nb == 2 ? tma_sum<2> : nb == 3 ? tma_sum<3> : nb == 4 ? tma_sum<4> : tma_sum<6>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
      const int64_t nboxes = rows / rb;
      for (int bpc : {16, 64}) {
        const int grid = (int)(nboxes / bpc);
        kern<<<grid, 256, smem>>>(tm, rb, rows, bpc, out);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) kern<<<grid, 256, smem>>>(tm, rb, rows, bpc, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("tma rows %2d NB %d (%2.0f KB in ring, %d CTA/SM) boxes/cta %2d: %.0f GB/s  %s\n", rb, nb,
               smem / 1024.0, per_sm, bpc, 3.0 * grid * bpc * bb / (ms * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
