// DMMA issue rate against the number of warps per SM sub-partition (development probe): one CTA per
// SM with 4*w warps (w per sub-partition), each warp issuing NT independent mma.sync.m8n8k4.f64
// accumulators in a loop; optionally an LDS pair per DMMA group (the GEMM consumer's fragment
// loads).  Answers: can ONE warp per sub-partition keep the FP64 tensor pipe busy?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_warps tools/dmma_warps.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NT, bool LDS>
__global__ void k(double* out, int iters) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i * 1e-3;
  __syncthreads();
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) c[t][0] = t, c[t][1] = -t;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    if (LDS) {  // 12 fragment loads per 32 DMMAs, as the 64 x 32 warp tile
      double f[12];
#pragma unroll
      for (int q = 0; q < 12; ++q) f[q] = sm[(q * 64 + lane + it) & 1023];
#pragma unroll
      for (int t = 0; t < NT; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[t][0]), "+d"(c[t][1])
                     : "d"(f[t % 8]), "d"(f[8 + t % 4]));
    } else {
#pragma unroll
      for (int t = 0; t < NT; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[t][0]), "+d"(c[t][1])
                     : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < NT; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NT, bool LDS>
void run(int sms, double* out, int w) {
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k<NT, LDS><<<sms, 128 * w>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  const double fma = (double)sms * 128 * w / 32 * iters * NT * 256.0;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"warps_per_subpartition\": %d, \"accumulators\": %d, \"lds\": %d, \"tflops\": %.3f, \"fma_per_clk_per_sm\": %.2f}\n",
         w, NT, (int)LDS, 2 * fma / (best * 1e-3) / 1e12, fma / (best * 1e-3) / (clk * 1e3) / sms);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 1024);
  for (int w : {1, 2, 4}) {
    run<32, false>(sms, out, w);
    run<32, true>(sms, out, w);
    run<16, false>(sms, out, w);
  }
  return 0;
}
