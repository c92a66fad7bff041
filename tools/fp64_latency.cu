// Dependent-chain latency of DADD, DMUL, DFMA, LDS and DMMA on one warp (clock64), for the
// small-problem path study:  nvcc -gencode arch=compute_100a,code=sm_100a
//   -O3 -o /tmp/fp64_latency tools/fp64_latency.cu && /tmp/fp64_latency
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double x0, double y0) {
  __shared__ double sh[64];
  const int t = threadIdx.x;
  sh[t] = x0 + t;
  __syncthreads();
  double x = x0, y = y0;
  long long c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = __dadd_rn(x, y);
  long long c1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = __dmul_rn(x, y);
  long long c2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = fma(x, y, y);
  long long c3 = clock64();
  int idx = t & 31;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) idx = (int)sh[idx] & 31;  // LDS -> F2I -> address chain
  long long c4 = clock64();
  double acc[2] = {x, y};
#pragma unroll 1
  for (int i = 0; i < 1024; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(acc[0]), "+d"(acc[1]) : "d"(x), "d"(y));
  long long c5 = clock64();
  out[t] = x + acc[0] + acc[1] + idx;
  if (t == 0) {
    cyc[0] = c1 - c0; cyc[1] = c2 - c1; cyc[2] = c3 - c2; cyc[3] = c4 - c3; cyc[4] = c5 - c4;
  }
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 64 * 8); cudaMallocManaged(&cyc, 5 * 8);
  lat<<<1, 32>>>(out, cyc, 1.0, 1e-300);
  cudaDeviceSynchronize();
  lat<<<1, 32>>>(out, cyc, 1.0, 1e-300);
  cudaDeviceSynchronize();
  const char* nm[5] = {"DADD", "DMUL", "DFMA", "LDS+F2I (address chain)", "DMMA.8x8x4 (accumulator chain)"};
  for (int i = 0; i < 5; ++i) printf("{\"op\": \"%s\", \"cycles_per_dependent_op\": %.1f}\n", nm[i], cyc[i] / 1024.0);
  return 0;
}
