// FP64 ceiling microbenchmark for sm_100a: DMMA (mma.sync f64 shapes) and DFMA issue rates.
// Used to derive the FP64 roofline denominator reported next to MEASURED_PEAKS.json (which has none).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int NT>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) { c[t][0] = t; c[t][1] = -t; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < NT; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < NT; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NT>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = (threadIdx.x + i) * 1e-3;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + (threadIdx.x + i) * 1e-4;
  double c[NT][4];
#pragma unroll
  for (int t = 0; t < NT; ++t) { c[t][0] = t; c[t][1] = -t; c[t][2] = 0; c[t][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < NT; ++t)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < NT; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NT>
__global__ void dfma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-7;
  double c[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) c[t] = t;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < NT; ++t) c[t] = fma(c[t], b, a);
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < NT; ++t) s += c[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
static double run(F kern, int blocks, int threads, int iters, double flop_per_warp_iter, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters);  // warm
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double warps = (double)blocks * threads / 32.0;
  return warps * iters * flop_per_warp_iter / (best * 1e-3) / 1e12;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clock(kHz attr) %d\n", p.name, p.multiProcessorCount, clk);
  double* out; CK(cudaMalloc(&out, 1 << 26));
  int sms = p.multiProcessorCount;
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2}) {
      double t1 = run(dmma_m8n8k4<8>, sms * bps, wpb * 32, iters, 8 * 2.0 * 8 * 8 * 4, out);
      double t2 = run(dmma_m8n8k4<16>, sms * bps, wpb * 32, iters / 2, 16 * 2.0 * 8 * 8 * 4, out);
      double t3 = run(dmma_m16n8k16<4>, sms * bps, wpb * 32, iters / 4, 4 * 2.0 * 16 * 8 * 16, out);
      double t4 = run(dfma_kernel<8>, sms * bps, wpb * 32, iters, 8 * 2.0 * 32, out);
      printf("warps/blk %2d blk/SM %d : DMMA m8n8k4 x8 %.2f TF  x16 %.2f TF | m16n8k16 x4 %.2f TF | DFMA x8 %.2f TF\n",
             wpb, bps, t1, t2, t3, t4);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
