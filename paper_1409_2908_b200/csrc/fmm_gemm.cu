// K2 / K4 / K5: grouped FP64 GEMM on the B200 FP64 tensor pipe.
//
// The leaf products M_l = alpha_l * S_l * T_l of the recursion ("Recursive calls ...
// compute M_r = S_r T_r"; the paper calls MKL dgemm there) and the classical peel strips
// run as ONE grouped launch: a task table {A, B, C, ld*, m, n, k, alpha, beta} and a
// prefix sum of CTA tiles; every CTA finds its task by binary search.
//
// sm_100a has no tcgen05 kind for f64 (ptxas rejects kind::f64), so the FP64 tensor path is the
// warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4; measured 37.1 TFLOP/s = 64 FMA/clk/SM at
// 1965 MHz, tools/fp64_peak.cu).  Operands are staged global -> shared by cp.async (LDGSTS,
// L2-only .cg) in a 4-stage pipeline, read into register fragments with conflict-free padded
// shared-memory layouts, and accumulated in registers: CTA tile 128x128x16, 8 warps of 64x32.
//
// Layout: all operands row-major (column-major problems are mapped to row-major by Prop. 1 in
// the planner).  Ragged edges are zero-filled by the cp.async src-size operand; 16-byte copies
// when every row start is 16-byte aligned, 8-byte copies otherwise.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include "fmm_internal.h"

namespace fmm {

namespace {
constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4, THREADS = 256;
constexpr int SA = BK + 4;  // A tile row stride in smem (doubles): conflict-free fragment reads
constexpr int SB = BN + 4;  // B tile row stride
constexpr int WM = 64, WN = 32;
constexpr int MI = WM / 8, NI = WN / 8;
constexpr int SMEM_A = BM * SA;  // doubles per stage
constexpr int SMEM_B = BK * SB;
constexpr size_t SMEM_BYTES = sizeof(double) * STAGES * (SMEM_A + SMEM_B);
constexpr int GROUP_M = 8;  // tile raster swizzle for L2 reuse

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(unsigned dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(unsigned dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <bool AL16>
__device__ __forceinline__ void load_stage(const GemmTask& t, double* As, double* Bs, int m0, int n0, int k0,
                                           int tid) {
  // A tile: BM rows x BK cols = BM*BK/2 16-byte chunks (4 per thread)
#pragma unroll
  for (int it = 0; it < (BM * BK / 2) / THREADS; ++it) {
    const int c = tid + it * THREADS;
    const int r = c / (BK / 2), kc = (c % (BK / 2)) * 2;
    const int gr = m0 + r, gk = k0 + kc;
    const double* src = t.A + (long long)gr * t.lda + gk;
    double* dst = As + r * SA + kc;
    const bool rok = gr < t.m;
    if (AL16) {
      int bytes = (rok && gk < t.k) ? 8 * min(2, t.k - gk) : 0;
      cp_async16(smem_u32(dst), bytes ? src : t.A, bytes);
    } else {
      cp_async8(smem_u32(dst), (rok && gk < t.k) ? src : t.A, (rok && gk < t.k) ? 8 : 0);
      cp_async8(smem_u32(dst + 1), (rok && gk + 1 < t.k) ? src + 1 : t.A, (rok && gk + 1 < t.k) ? 8 : 0);
    }
  }
  // B tile: BK rows x BN cols
#pragma unroll
  for (int it = 0; it < (BK * BN / 2) / THREADS; ++it) {
    const int c = tid + it * THREADS;
    const int r = c / (BN / 2), nc = (c % (BN / 2)) * 2;
    const int gk = k0 + r, gn = n0 + nc;
    const double* src = t.B + (long long)gk * t.ldb + gn;
    double* dst = Bs + r * SB + nc;
    const bool rok = gk < t.k;
    if (AL16) {
      int bytes = (rok && gn < t.n) ? 8 * min(2, t.n - gn) : 0;
      cp_async16(smem_u32(dst), bytes ? src : t.B, bytes);
    } else {
      cp_async8(smem_u32(dst), (rok && gn < t.n) ? src : t.B, (rok && gn < t.n) ? 8 : 0);
      cp_async8(smem_u32(dst + 1), (rok && gn + 1 < t.n) ? src + 1 : t.B, (rok && gn + 1 < t.n) ? 8 : 0);
    }
  }
}

template <bool AL16>
__global__ void __launch_bounds__(THREADS, 1)
    grouped_dgemm(const GemmTask* __restrict__ tasks, int ntasks) {
  extern __shared__ __align__(128) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * SMEM_A;

  // ---- find this CTA's task (binary search on tile_begin) and tile ----
  const int bid = blockIdx.x;
  int lo = 0, hi = ntasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tasks[mid].tile_begin <= bid) lo = mid; else hi = mid - 1;
  }
  const GemmTask t = tasks[lo];
  const int local = bid - t.tile_begin;
  const int span = GROUP_M * t.tiles_n;
  const int group = local / span;
  const int first_m = group * GROUP_M;
  const int gsize = min(t.tiles_m - first_m, GROUP_M);
  const int tm = first_m + (local % span) % gsize;
  const int tn = (local % span) / gsize;
  const int m0 = tm * BM, n0 = tn * BN;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp / (BN / WN)) * WM, wn = (warp % (BN / WN)) * WN;

  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int KT = (t.k + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage<AL16>(t, As + s * SMEM_A, Bs + s * SMEM_B, m0, n0, s * BK, tid);
    cp_commit();
  }

  const int ar = wm + (lane >> 2), ac = lane & 3;  // A fragment: row lane/4, col lane%4
  const int br = lane & 3, bc = wn + (lane >> 2);  // B fragment: row lane%4, col lane/4
  for (int kt = 0; kt < KT; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    const int nk = kt + STAGES - 1;
    if (nk < KT) load_stage<AL16>(t, As + (nk % STAGES) * SMEM_A, Bs + (nk % STAGES) * SMEM_B, m0, n0, nk * BK, tid);
    cp_commit();
    const double* as = As + (kt % STAGES) * SMEM_A;
    const double* bs = Bs + (kt % STAGES) * SMEM_B;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[MI], b[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = as[(ar + i * 8) * SA + kk + ac];
#pragma unroll
      for (int j = 0; j < NI; ++j) b[j] = bs[(kk + br) * SB + bc + j * 8];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma(acc[i][j], a[i], b[j]);
    }
  }
  cp_wait<0>();

  // ---- epilogue: C = alpha * acc (+ beta * C) ----
  const double alpha = t.alpha, beta = t.beta;
  const bool vec_ok = AL16 && ((t.ldc & 1) == 0) && ((reinterpret_cast<uintptr_t>(t.C) & 15) == 0);
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int row = m0 + wm + i * 8 + (lane >> 2);
    if (row >= t.m) continue;
    double* crow = t.C + (long long)row * t.ldc;
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const int col = n0 + wn + j * 8 + (lane & 3) * 2;
      double v0 = alpha * acc[i][j][0], v1 = alpha * acc[i][j][1];
      if (vec_ok && col + 1 < t.n) {
        double2* p = reinterpret_cast<double2*>(crow + col);
        if (beta != 0.0) {
          const double2 o = *p;
          v0 = fma(beta, o.x, v0);
          v1 = fma(beta, o.y, v1);
        }
        *p = make_double2(v0, v1);
      } else {
        if (col < t.n) crow[col] = beta != 0.0 ? fma(beta, crow[col], v0) : v0;
        if (col + 1 < t.n) crow[col + 1] = beta != 0.0 ? fma(beta, crow[col + 1], v1) : v1;
      }
    }
  }
}
}  // namespace

int gemm_tile_m() { return BM; }
int gemm_tile_n() { return BN; }

long long gemm_prepare(std::vector<GemmTask>& tasks, int bm, int bn) {
  long long total = 0;
  for (auto& t : tasks) {
    t.tiles_m = (t.m + bm - 1) / bm;
    t.tiles_n = (t.n + bn - 1) / bn;
    t.tile_begin = (int)total;
    total += (long long)t.tiles_m * t.tiles_n;
  }
  if (total > 0x7fffffffLL) throw Error(FMM_E_UNSUPPORTED, "too many GEMM tiles in one launch");
  return total;
}

void gemm_uniform_grid(const std::vector<GemmTask>& tasks, int* tm, int* tn) {
  *tm = *tn = 0;
  if (tasks.empty()) return;
  for (const auto& t : tasks)
    if (t.tiles_m != tasks[0].tiles_m || t.tiles_n != tasks[0].tiles_n) return;
  *tm = tasks[0].tiles_m;
  *tn = tasks[0].tiles_n;
}

bool gemm_tasks_aligned16(const std::vector<GemmTask>& tasks) {
  for (const auto& t : tasks) {
    if ((reinterpret_cast<uintptr_t>(t.A) & 15) || (reinterpret_cast<uintptr_t>(t.B) & 15)) return false;
    if ((t.lda & 1) || (t.ldb & 1)) return false;
  }
  return true;
}

void gemm_launch(const GemmTask* d_tasks, int ntasks, long long total_tiles, bool aligned16, cudaStream_t stream) {
  if (total_tiles <= 0 || ntasks <= 0) return;
  static std::atomic<unsigned long long> configured{0};  // bit d: attribute set on device d
  int dev_ = 0;
  FMM_CUDA(cudaGetDevice(&dev_));
  const unsigned long long bit = 1ull << (dev_ & 63);
  if (!(configured.load() & bit)) {
    FMM_CUDA(cudaFuncSetAttribute(grouped_dgemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
    FMM_CUDA(cudaFuncSetAttribute(grouped_dgemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
    configured.fetch_or(bit);
  }
  if (aligned16)
    grouped_dgemm<true><<<(unsigned)total_tiles, THREADS, SMEM_BYTES, stream>>>(d_tasks, ntasks);
  else
    grouped_dgemm<false><<<(unsigned)total_tiles, THREADS, SMEM_BYTES, stream>>>(d_tasks, ntasks);
  FMM_CUDA(cudaGetLastError());
}

}  // namespace fmm
