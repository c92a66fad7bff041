// Per-SM read+write bandwidth of an addition-CTA-like pipeline: k CTAs (one per SM, 384 threads),
// warp 0 lane 0 streams CH-byte chunks of the CTA's slice into an NS-stage shared-memory ring with
// 1-D bulk copies; warps 1..11 read each stage (16-byte LDS per thread) and store it to a
// destination slice (16-byte STG, OUTX copies of the input bytes: the output streams of a formation).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c)); }
__device__ __forceinline__ void mbar_wait(unsigned b, unsigned ph) {
  asm volatile("{ .reg .pred q; W: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W; }" ::"r"(b), "r"(ph) : "memory");
}

template <int CH, int NS, int OUTX>
__global__ void __launch_bounds__(384, 1) ring(const char* __restrict__ src, char* __restrict__ dst, size_t per_cta) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm + NS * CH);
  const unsigned full0 = smem_u32(bars), empty0 = full0 + 8 * NS;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(full0 + 8 * s, 1), mbar_init(empty0 + 8 * s, 11);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const char* p = src + blockIdx.x * per_cta;
  char* q = dst + blockIdx.x * per_cta * OUTX;
  const size_t n = per_cta / CH;
  if (warp == 0) {
    if (lane == 0) {
      for (size_t c = 0; c < n; ++c) {
        const int s = c % NS;
        const unsigned ph = (c / NS) & 1;
        mbar_wait(empty0 + 8 * s, ph ^ 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full0 + 8 * s), "r"(CH) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm) + s * CH),
                     "l"(p + c * CH), "r"(CH), "r"(full0 + 8 * s) : "memory");
      }
    }
    return;
  }
  const int t = threadIdx.x - 32;  // 0..351
  for (size_t c = 0; c < n; ++c) {
    const int s = c % NS;
    mbar_wait(full0 + 8 * s, (c / NS) & 1);
    const double2* in = reinterpret_cast<const double2*>(sm + s * CH);
    for (int i = t; i < CH / 16; i += 352) {
      const double2 v = in[i];
#pragma unroll
      for (int o = 0; o < OUTX; ++o) {
        double2 w = make_double2(v.x + o, v.y - o);
        *reinterpret_cast<double2*>(q + (c * CH) * OUTX + o * CH + i * 16) = w;
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8 * s) : "memory");
  }
}

// the same, but the compute warps write the output chunk into shared memory and warp 0 lane 1
// stores it with a 1-D bulk copy (cp.async.bulk.global.shared::cta, bulk-group completion)
template <int CH, int NS>
__global__ void __launch_bounds__(384, 1) ring_tma_store(const char* __restrict__ src, char* __restrict__ dst, size_t per_cta) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* out = sm + NS * CH;  // NS output stages
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm + 2 * NS * CH);
  const unsigned full0 = smem_u32(bars), empty0 = full0 + 8 * NS, done0 = empty0 + 8 * NS, oempty0 = done0 + 8 * NS;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(full0 + 8 * s, 1), mbar_init(empty0 + 8 * s, 11), mbar_init(done0 + 8 * s, 11), mbar_init(oempty0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const char* p = src + blockIdx.x * per_cta;
  char* q = dst + blockIdx.x * per_cta;
  const size_t n = per_cta / CH;
  if (warp == 0) {
    if (lane == 0) {
      for (size_t c = 0; c < n; ++c) {
        const int s = c % NS;
        const unsigned ph = (c / NS) & 1;
        mbar_wait(empty0 + 8 * s, ph ^ 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full0 + 8 * s), "r"(CH) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm) + s * CH),
                     "l"(p + c * CH), "r"(CH), "r"(full0 + 8 * s) : "memory");
      }
    } else if (lane == 1) {
      for (size_t c = 0; c < n; ++c) {
        const int s = c % NS;
        mbar_wait(done0 + 8 * s, (c / NS) & 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(q + c * CH), "r"(smem_u32(out) + s * CH), "r"(CH) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NS - 2) : "memory");
        // the store NS-2 groups back has read its shared memory: release that output stage
        if (c >= NS - 2) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)(oempty0 + 8 * ((c - (NS - 2)) % NS))) : "memory");
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    return;
  }
  const int t = threadIdx.x - 32;
  for (size_t c = 0; c < n; ++c) {
    const int s = c % NS;
    mbar_wait(full0 + 8 * s, (c / NS) & 1);
    if (c >= NS) mbar_wait(oempty0 + 8 * s, ((c - NS) / NS) & 1);
    const double2* in = reinterpret_cast<const double2*>(sm + s * CH);
    double2* o = reinterpret_cast<double2*>(out + s * CH);
    for (int i = t; i < CH / 16; i += 352) {
      const double2 v = in[i];
      o[i] = make_double2(v.x + 1, v.y - 1);
    }
    __syncwarp();
    if (lane == 0) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8 * s) : "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(done0 + 8 * s) : "memory");
    }
  }
}

template <int CH, int NS>
void run_tma(const char* src, char* dst, int k, size_t per, cudaEvent_t e0, cudaEvent_t e1) {
  const int smem = 2 * NS * CH + 32 * NS + 64;
  cudaFuncSetAttribute(ring_tma_store<CH, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  ring_tma_store<CH, NS><<<k, 384, smem>>>(src, dst, per);
  cudaEventRecord(e0);
  ring_tma_store<CH, NS><<<k, 384, smem>>>(src, dst, per);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)per * k * 2;
  printf("k=%3d CH=%6d NS=%d TMA store: %8.1f GB/s (%6.1f /SM, read+write)  %s\n", k, CH, NS, bytes / (ms * 1e-3) / 1e9,
         bytes / (ms * 1e-3) / 1e9 / k, cudaGetErrorString(cudaGetLastError()));
}

template <int CH, int NS, int OUTX>
void run(const char* src, char* dst, int k, size_t per, cudaEvent_t e0, cudaEvent_t e1) {
  const int smem = NS * CH + 16 * NS + 64;
  cudaFuncSetAttribute(ring<CH, NS, OUTX>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  ring<CH, NS, OUTX><<<k, 384, smem>>>(src, dst, per);
  cudaEventRecord(e0);
  ring<CH, NS, OUTX><<<k, 384, smem>>>(src, dst, per);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)per * k * (1 + OUTX);
  printf("k=%3d CH=%6d NS=%d OUTX=%d: %8.1f GB/s (%6.1f /SM, read+write)  %s\n", k, CH, NS, OUTX, bytes / (ms * 1e-3) / 1e9,
         bytes / (ms * 1e-3) / 1e9 / k, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const size_t per = 24ull << 20;  // bytes read per CTA
  char *src, *dst;
  cudaMalloc(&src, per * 148);
  cudaMalloc(&dst, per * 148 * 2);
  cudaMemset(src, 0, per * 148);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int k : {4, 16}) {
    run<16384, 12, 1>(src, dst, k, per, e0, e1);
    run<32768, 6, 1>(src, dst, k, per, e0, e1);
    run<16384, 12, 2>(src, dst, k, per, e0, e1);
    run<8192, 24, 1>(src, dst, k, per, e0, e1);
    run_tma<16384, 6>(src, dst, k, per, e0, e1);
    run_tma<8192, 12>(src, dst, k, per, e0, e1);
  }
  return 0;
}
