// FP32 / FP64 / packed-FP32x2 issue-rate microbenchmark: independent FMA chains, CUDA-event timed.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T, int CH>
__global__ void chain(T* out, int iters, T a, T b) {
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
__global__ void chain_f2(float* out, int iters, float a, float b) {
  float2 x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = make_float2(threadIdx.x + c, c);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      unsigned long long r, xv = *reinterpret_cast<unsigned long long*>(&x[c]);
      float2 av = make_float2(a, a), bv = make_float2(b, b);
      unsigned long long aa = *reinterpret_cast<unsigned long long*>(&av), bb = *reinterpret_cast<unsigned long long*>(&bv);
      asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(xv), "l"(aa), "l"(bb));
      x[c] = *reinterpret_cast<float2*>(&r);
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c].x + x[c].y;
  if (s == 12345.678f) out[0] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s sms %d l2 %d smem/block optin %zu clock %d kHz\n", p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, p.clockRate);
  void* buf; cudaMalloc(&buf, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    chain<float, 8><<<blocks, threads>>>((float*)buf, iters, 1.0001f, 0.5f);
    cudaEventRecord(e0); chain<float, 8><<<blocks, threads>>>((float*)buf, iters, 1.0001f, 0.5f); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double f32 = 2.0 * blocks * threads * 8.0 * iters / (ms * 1e-3) / 1e12;
    cudaEventRecord(e0); chain<double, 8><<<blocks, threads>>>((double*)buf, iters / 4, 1.0001, 0.5); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double f64 = 2.0 * blocks * threads * 8.0 * (iters / 4) / (ms * 1e-3) / 1e12;
    cudaEventRecord(e0); chain_f2<<<blocks, threads>>>((float*)buf, iters, 1.0001f, 0.5f); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double f2 = 4.0 * blocks * threads * 8.0 * iters / (ms * 1e-3) / 1e12;
    printf("rep %d: fp32 FFMA %.1f TFLOP/s  fp64 DFMA %.1f TFLOP/s  f32x2 FFMA2 %.1f TFLOP/s  (%s)\n", rep, f32, f64, f2, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
