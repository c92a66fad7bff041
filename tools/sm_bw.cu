// Per-SM read bandwidth probe: k CTAs (one per SM, 384 threads, ~200 KB smem), each streaming its
// own disjoint slice of a large buffer (a) with LDG.128 (12 warps, U loads in flight per lane) or
// (b) with 1-D bulk copies (TMA engine) into a ring of shared-memory buffers.  Prints GB/s per SM.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int U>
__global__ void __launch_bounds__(384, 1) ldg_read(const double2* __restrict__ src, size_t per_cta, double* out) {
  const double2* p = src + blockIdx.x * per_cta;
  double acc = 0;
  for (size_t i = threadIdx.x; i < per_cta; i += 384 * U) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t j = i + (size_t)u * 384;
      v[u] = j < per_cta ? __ldcg(p + j) : make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
  }
  if (acc == 12345.678) out[0] = acc;
}

// bulk: warp w of the CTA streams chunks of CH bytes through NB buffers
template <int CH, int NB>
__global__ void __launch_bounds__(384, 1) bulk_read(const char* __restrict__ src, size_t per_cta, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = 12;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm + nw * NB * CH);
  const unsigned buf0 = smem_u32(sm) + warp * NB * CH;
  const unsigned bar0 = smem_u32(bars) + warp * NB * 8;
  if (lane == 0)
    for (int b = 0; b < NB; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * b));
  __syncwarp();
  const char* p = src + blockIdx.x * per_cta + (size_t)warp * (per_cta / nw);
  const size_t n = per_cta / nw / CH;
  double acc = 0;
  unsigned phase = 0;
  auto issue = [&](size_t c) {
    const int b = c % NB;
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar0 + 8 * b), "r"(CH) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(buf0 + b * CH),
                   "l"(p + c * CH), "r"(CH), "r"(bar0 + 8 * b) : "memory");
    }
  };
  for (size_t c = 0; c < NB && c < n; ++c) issue(c);
  for (size_t c = 0; c < n; ++c) {
    const int b = c % NB;
    asm volatile("{ .reg .pred q; W: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W; }" ::"r"(bar0 + 8 * b),
                 "r"((phase >> b) & 1) : "memory");
    phase ^= 1u << b;
    const double2* s = reinterpret_cast<const double2*>(sm + warp * NB * CH + b * CH);
    for (int i = lane; i < CH / 16; i += 32) acc += s[i].x;
    __syncwarp();
    if (c + NB < n) issue(c + NB);
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  const size_t total = 8ull << 30;  // 8 GB
  char* buf;
  double* out;
  cudaMalloc(&buf, total);
  cudaMalloc(&out, 8);
  cudaMemset(buf, 0, total);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int ks[] = {1, 2, 4, 8, 16, 148};
  for (int k : ks) {
    const size_t per = (total / 148) / (12 * 65536) * (12 * 65536);  // bytes per CTA (fixed per-CTA work)
    float ms;
    // LDG
    ldg_read<4><<<k, 384>>>((const double2*)buf, per / 16, out);
    cudaEventRecord(e0);
    ldg_read<4><<<k, 384>>>((const double2*)buf, per / 16, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double ldg = per * 1.0 * k / (ms * 1e-3) / 1e9;
    ldg_read<8><<<k, 384>>>((const double2*)buf, per / 16, out);
    cudaEventRecord(e0);
    ldg_read<8><<<k, 384>>>((const double2*)buf, per / 16, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double ldg8 = per * 1.0 * k / (ms * 1e-3) / 1e9;
    // bulk
    constexpr int CH = 8192, NB = 2;
    const int smem = 12 * NB * CH + 12 * NB * 8;
    cudaFuncSetAttribute(bulk_read<CH, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    bulk_read<CH, NB><<<k, 384, smem>>>(buf, per, out);
    cudaEventRecord(e0);
    bulk_read<CH, NB><<<k, 384, smem>>>(buf, per, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double bulk = per * 1.0 * k / (ms * 1e-3) / 1e9;
    constexpr int CH2 = 4096, NB2 = 4;
    const int smem2 = 12 * NB2 * CH2 + 12 * NB2 * 8;
    cudaFuncSetAttribute(bulk_read<CH2, NB2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    bulk_read<CH2, NB2><<<k, 384, smem2>>>(buf, per, out);
    cudaEventRecord(e0);
    bulk_read<CH2, NB2><<<k, 384, smem2>>>(buf, per, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double bulk2 = per * 1.0 * k / (ms * 1e-3) / 1e9;
    printf("k=%3d  LDG.128 x4: %7.1f GB/s (%6.1f /SM)  x8: %7.1f (%6.1f /SM)  bulk 2x8KB: %7.1f (%6.1f /SM)  bulk 4x4KB: %7.1f (%6.1f /SM)  err=%s\n",
           k, ldg, ldg / k, ldg8, ldg8 / k, bulk, bulk / k, bulk2, bulk2 / k, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
