// FP32 / FP64 FMA-rate probe for bench.py's roofline peaks (measured in the
// same run as the kernels they rate): independent FMA chains over 8 CTAs per
// SM, CUDA-event timed, best of three.  Measurement infrastructure, not part
// of the product library.
#include <cuda_runtime.h>

template <typename T, int CH>
__global__ void fma_chain(T* out, int iters, T a, T b) {
  T x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = (T)(threadIdx.x + c);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = x[c] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == (T)12345.678) out[0] = s;
}

// kind 0: FP32 FFMA, 1: FP64 DFMA.  Returns TFLOP/s (2 flops per FMA), < 0 on error.
extern "C" double ct_probe_fma_tflops(int kind) {
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, 0) != cudaSuccess) return -1.0;
  void* buf = nullptr;
  if (cudaMalloc(&buf, 64) != cudaSuccess) return -1.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = p.multiProcessorCount * 8, threads = 256;
  const int iters = kind == 0 ? 4096 : 1024;
  double best = 0.0;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    if (kind == 0)
      fma_chain<float, 16><<<blocks, threads>>>((float*)buf, iters, 1.0001f, 0.5f);
    else
      fma_chain<double, 16><<<blocks, threads>>>((double*)buf, iters, 1.0001, 0.5);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = 2.0 * blocks * threads * 16.0 * iters / (ms * 1e-3) / 1e12;
    if (rep > 0 && tf > best) best = tf;  // rep 0 warms the clocks
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  return cudaGetLastError() == cudaSuccess ? best : -1.0;
}
