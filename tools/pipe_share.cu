// Does FP64 ALU work (DADD) beside DMMA slow either down?  One CTA per SM, 8 "tensor" warps
// issuing independent mma.sync.m8n8k4.f64 from registers, 4 "alu" warps issuing independent DADD
// chains; each role timed alone and together (clock64 per warp, max over warps).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(384, 1) kern(int mode, int iters, double* out, unsigned long long* cyc) {
  const int warp = threadIdx.x >> 5;
  const bool tensor = warp >= 4;
  const bool run = (mode == 2) || (mode == 0 && tensor) || (mode == 1 && !tensor);
  double r = 0;
  unsigned long long t0 = clock64();
  if (run && tensor) {
    double acc[8][2] = {};
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma(acc[j], a, b);
    }
    for (int j = 0; j < 8; ++j) r += acc[j][0] + acc[j][1];
  } else if (run) {
    double x[8];
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
    const double y = 1e-9 * threadIdx.x;
    for (int i = 0; i < iters * 4; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = __dadd_rn(x[j], y);
    }
    for (int j = 0; j < 8; ++j) r += x[j];
  }
  unsigned long long t1 = clock64();
  if (r == 1.2345) out[0] = r;
  if ((threadIdx.x & 31) == 0 && run) atomicMax(&cyc[tensor ? 0 : 1], t1 - t0);
}

int main() {
  double* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 16);
  const int iters = 20000;
  const char* names[] = {"DMMA warps alone", "DADD warps alone", "both together"};
  for (int mode = 0; mode < 3; ++mode) {
    unsigned long long h[2] = {0, 0};
    kern<<<148, 384>>>(mode, iters, out, cyc);  // warm
    cudaMemset(cyc, 0, 16);
    kern<<<148, 384>>>(mode, iters, out, cyc);
    cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
    // per SM: DMMA 8 warps * iters * 8 * 256 FMA; DADD 4 warps * 32 lanes * iters*4*8 adds
    const double dmma_fma_per_clk = h[0] ? 8.0 * iters * 8 * 256 / h[0] : 0;
    const double dadd_per_clk = h[1] ? 4.0 * 32 * iters * 4 * 8 / h[1] : 0;
    printf("%-18s: DMMA warps %10llu clk (%.1f FMA/clk/SM)   DADD warps %10llu clk (%.1f DADD/clk/SM)  %s\n", names[mode],
           h[0], dmma_fma_per_clk, h[1], dadd_per_clk, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
