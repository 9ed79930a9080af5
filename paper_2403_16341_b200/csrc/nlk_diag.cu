// Diagnostics: the measured FP64 (and FP32) FMA-pipe peaks used as the
// roofline denominators (MEASURED_PEAKS.json carries only HBM and bf16
// figures).  Each thread runs 8 independent FMA chains; FLOPs = 2 * 8 * iters
// per thread.
#include <cuda_runtime.h>

#include <string>

#include "nlk_b200.h"

namespace {
template <class T>
__global__ void __launch_bounds__(256) fma_chains(T* sink, long long iters, T a) {
  T x0 = threadIdx.x * T(1e-3), x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  T x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  const T b = T(1e-7);
#pragma unroll 4
  for (long long i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  T s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (s == T(12345.678)) sink[0] = s;  // keeps the chains alive
}
thread_local std::string g_diag_err;
}  // namespace

template <class T>
int fma_peak(int64_t iters, double* tflops_out, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return NLK_ERR_CUDA;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  T* sink = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&sink), sizeof(T), s) != cudaSuccess) return NLK_ERR_CUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  fma_chains<T><<<blocks, threads, 0, s>>>(sink, iters / 8, T(0.999999));  // warm-up
  cudaEventRecord(e0, s);
  fma_chains<T><<<blocks, threads, 0, s>>>(sink, iters, T(0.999999));
  cudaEventRecord(e1, s);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(sink, s);
  if (e != cudaSuccess) return NLK_ERR_CUDA;
  const double flops = 2.0 * 8.0 * static_cast<double>(iters) * blocks * threads;
  if (tflops_out) *tflops_out = flops / (ms * 1e-3) / 1e12;
  return NLK_OK;
}

extern "C" NLK_API int nlk_fp64_peak(int64_t iters, double* tflops_out, void* stream) {
  return fma_peak<double>(iters, tflops_out, stream);
}
extern "C" NLK_API int nlk_fp32_peak(int64_t iters, double* tflops_out, void* stream) {
  return fma_peak<float>(iters, tflops_out, stream);
}
