// FP64 ceiling probe: the roofline denominator of the leaf GEMM, measured in-run (the same
// kernels as tools/fp64_peak.cu).  DMMA: independent mma.sync.m8n8k4.f64 accumulators per warp;
// DFMA: independent fma chains.  Launched with 8 warps x 2 CTAs per SM.
#include <cuda_runtime.h>

#include "fmm_internal.h"

namespace {
constexpr int NT = 16;
__global__ void probe_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) c[t][0] = t, c[t][1] = -t;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < NT; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < NT; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void probe_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-7;
  double c[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) c[t] = t;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t] = fma(c[t], b, a);
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace

extern "C" fmm_status_t fmm_probe_fp64_peak(double* dmma_tflops, double* dfma_tflops) {
  FMM_API_BEGIN
  int dev = 0, sms = 0;
  FMM_CUDA(cudaGetDevice(&dev));
  FMM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int blocks = 2 * sms, threads = 256;
  double* out = nullptr;
  FMM_CUDA(cudaMalloc(&out, sizeof(double) * blocks * threads));
  cudaEvent_t e0, e1;
  FMM_CUDA(cudaEventCreate(&e0));
  FMM_CUDA(cudaEventCreate(&e1));
  auto best_ms = [&](auto kern, int iters) {
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      FMM_CUDA(cudaEventRecord(e0, 0));
      kern<<<blocks, threads>>>(out, iters);
      FMM_CUDA(cudaEventRecord(e1, 0));
      FMM_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      FMM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      if (rep > 0 && ms < best) best = ms;  // rep 0 is the warm-up
    }
    return (double)best;
  };
  const double warps = blocks * threads / 32.0;
  const int it_m = 4000, it_f = 20000;
  const double tm = best_ms(probe_dmma, it_m);
  const double tf = best_ms(probe_dfma, it_f);
  if (dmma_tflops) *dmma_tflops = warps * it_m * NT * (2.0 * 8 * 8 * 4) / (tm * 1e-3) / 1e12;
  if (dfma_tflops) *dfma_tflops = warps * it_f * 8 * (2.0 * 32) / (tf * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return FMM_OK;
  FMM_API_END
}
