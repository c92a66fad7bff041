// K4: thin peel strips (SPEC S:290 (b) last P-P' rows, (c) last N-N' columns).
//
// A strip is a classical product with one tiny dimension (1 to 2N-1 rows or columns).  On the
// 128-row DMMA tile it would waste up to 99 % of the tensor work, so thin tasks of a strip launch
// run here instead, on the FP64 CUDA cores, HBM/L2-bound:
//   row strips (m <= 8): a block covers 128 output columns x 4 k-slices, a thread a column pair
//       (16-byte loads of B, so two warps read 1 KB of a B row at a time), two batches of four
//       B rows in flight per thread; each thread keeps all m rows of its columns in registers
//       over its k-slice (B read once, coalesced; A[i][k] a warp-uniform broadcast), and the
//       slices are reduced in order through shared memory.  The round-1 form (32 columns x 8
//       k-slices, 256-byte row segments) stays selectable (FMM_SKINNY_ROWS=narrow): on c3 the
//       row strips take 88 against 195 us (ncu), all strips 0.23 against 0.34 ms (events).
//   column strips (n <= 8): two output rows per warp; lanes split k (A rows read coalesced,
//       16-byte loads), the B strip is staged transposed in shared memory per k-chunk (padded
//       stride: conflict-free stores; 16-byte conflict-free loads), each lane accumulates all n
//       outputs, then a warp shuffle reduction.
// C = alpha * A B + beta * C, same task table as the GEMM kernels.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "fmm_internal.h"

namespace fmm {

namespace {
constexpr int THIN = 8;  // strips are < 2 x (base-case dim) wide

// 32 columns x 8 k-slices per block: each thread sums k = ks, ks+8, ... for its column and all
// m rows (independent loads in flight across slices), then the slices are reduced in smem.
// TH: the launch's largest strip height rounded up to a power of two (1, 2, 4 or 8): the
// accumulators of rows that cannot occur take no registers, so thin strips run at a higher
// occupancy with more loads in flight
template <int TH>
__global__ void __launch_bounds__(256) skinny_rows(const GemmTask* __restrict__ tasks, const int* __restrict__ ids,
                                                   int count) {
  __shared__ double red[8][TH][33];
  const GemmTask t = tasks[ids[blockIdx.y]];
  const int tx = threadIdx.x & 31, ks = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + tx;
  double acc[TH];
#pragma unroll
  for (int i = 0; i < TH; ++i) acc[i] = 0.0;
  if (j < t.n) {
    int k = ks;
#ifndef FMM_SKINNY_ROW_UNROLL
#define FMM_SKINNY_ROW_UNROLL 8  // measured on c3: 4 -> 8 in flight, strips 0.372 -> 0.349 ms
#endif
    constexpr int U = TH <= 2 ? 2 * FMM_SKINNY_ROW_UNROLL : FMM_SKINNY_ROW_UNROLL;
    for (; k + 8 * (U - 1) < t.k; k += 8 * U) {  // U independent B loads in flight per thread
      double b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) b[u] = __ldg(t.B + (long long)(k + 8 * u) * t.ldb + j);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < TH; ++i)
          if (i < t.m) acc[i] = fma(__ldg(t.A + (long long)i * t.lda + k + 8 * u), b[u], acc[i]);
    }
    for (; k < t.k; k += 8) {
      const double b = __ldg(t.B + (long long)k * t.ldb + j);
#pragma unroll
      for (int i = 0; i < TH; ++i)
        if (i < t.m) acc[i] = fma(__ldg(t.A + (long long)i * t.lda + k), b, acc[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < TH; ++i) red[ks][i][tx] = acc[i];
  __syncthreads();
  // thread (ks, tx) finalises row i = ks of column j
  if (j < t.n) {
#pragma unroll
    for (int h = 0; h < 1; ++h) {
      const int i = ks + 8 * h;
      if (i < t.m && i < TH) {
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) v += red[q][i][tx];
        double* c = t.C + (long long)i * t.ldc + j;
        *c = t.beta != 0.0 ? fma(t.beta, *c, t.alpha * v) : t.alpha * v;
      }
    }
  }
}

// Row strips, wide-segment form (the default): a block covers 128 output columns x 4 k-slices;
// each thread owns a column pair (16-byte loads of B), so the two warps of a slice read 1 KB of a
// B row at a time instead of 256 bytes (fewer DRAM pages open per byte; round 2, DESIGN.md
// sec. 6), eight rows in flight per thread; slices reduced in order through shared memory.
template <int TH>
__global__ void __launch_bounds__(256) skinny_rows_w(const GemmTask* __restrict__ tasks, const int* __restrict__ ids,
                                                     int count) {
#ifndef FMM_SKINNY_ROWW_U
#define FMM_SKINNY_ROWW_U 4  // rows per batch (two batches in flight)
#endif
  constexpr int KSL = 4, U = FMM_SKINNY_ROWW_U;
  __shared__ double2 red[KSL][TH][64];
  const GemmTask t = tasks[ids[blockIdx.y]];
  const int tx = threadIdx.x & 63, ks = threadIdx.x >> 6;
  const int j = blockIdx.x * 128 + 2 * tx;
  const bool two = j + 1 < t.n;
  const bool v2 = two && ((reinterpret_cast<uintptr_t>(t.B) & 15) == 0) && ((t.ldb & 1) == 0);
  double2 acc[TH];
#pragma unroll
  for (int i = 0; i < TH; ++i) acc[i] = make_double2(0.0, 0.0);
  auto ldb2 = [&](int k) -> double2 {
    const double* p = t.B + (long long)k * t.ldb + j;
    if (v2) return __ldg(reinterpret_cast<const double2*>(p));
    return make_double2(__ldg(p), two ? __ldg(p + 1) : 0.0);
  };
  if (j < t.n) {
    int k = ks;
    // software-pipelined: the next batch of U rows is in flight while this one is summed
    const int kfull = t.k - KSL * (U - 1);  // batches starting below kfull are whole
    double2 b[U];
    if (k < kfull) {
#pragma unroll
      for (int u = 0; u < U; ++u) b[u] = ldb2(k + KSL * u);
    }
    for (; k < kfull; k += KSL * U) {
      double2 nb[U];
      const bool more = k + KSL * U < kfull;
      if (more) {
#pragma unroll
        for (int u = 0; u < U; ++u) nb[u] = ldb2(k + KSL * U + KSL * u);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < TH; ++i)
          if (i < t.m) {
            const double a = __ldg(t.A + (long long)i * t.lda + k + KSL * u);
            acc[i].x = fma(a, b[u].x, acc[i].x);
            acc[i].y = fma(a, b[u].y, acc[i].y);
          }
      if (more) {
#pragma unroll
        for (int u = 0; u < U; ++u) b[u] = nb[u];
      }
    }
    for (; k < t.k; k += KSL) {
      const double2 b = ldb2(k);
#pragma unroll
      for (int i = 0; i < TH; ++i)
        if (i < t.m) {
          const double a = __ldg(t.A + (long long)i * t.lda + k);
          acc[i].x = fma(a, b.x, acc[i].x);
          acc[i].y = fma(a, b.y, acc[i].y);
        }
    }
  }
#pragma unroll
  for (int i = 0; i < TH; ++i) red[ks][i][tx] = acc[i];
  __syncthreads();
  if (j < t.n) {
    for (int i = ks; i < TH && i < t.m; i += KSL) {
      double2 v = red[0][i][tx];
#pragma unroll
      for (int q = 1; q < KSL; ++q) v.x += red[q][i][tx].x, v.y += red[q][i][tx].y;
      double* c = t.C + (long long)i * t.ldc + j;
      c[0] = t.beta != 0.0 ? fma(t.beta, c[0], t.alpha * v.x) : t.alpha * v.x;
      if (two) c[1] = t.beta != 0.0 ? fma(t.beta, c[1], t.alpha * v.y) : t.alpha * v.y;
    }
  }
}

// Column strips: 16 rows per block (2 per warp); the B strip (k x n, n <= 8) is staged transposed
// through shared memory in k-chunks; lanes split k and read A rows coalesced, 16 bytes at a time
// when A is 16-byte aligned with an even lda, with up to 16 loads in flight per lane; each lane
// accumulates all n outputs of its rows, then a warp shuffle reduction.
#ifndef FMM_SKINNY_RPW
#define FMM_SKINNY_RPW 2
#endif
#ifndef FMM_SKINNY_KC
#define FMM_SKINNY_KC 256
#endif
constexpr int ROWS_PER_WARP = FMM_SKINNY_RPW;
#ifndef FMM_SKINNY_COLS_MINB
#define FMM_SKINNY_COLS_MINB 4  // blocks per SM the register budget must allow (80 -> 64 registers)
#endif
template <int TH>
__global__ void __launch_bounds__(256, TH <= 4 ? FMM_SKINNY_COLS_MINB : 3) skinny_cols(const GemmTask* __restrict__ tasks, const int* __restrict__ ids,
                                                   int count) {
  // k-chunk of the staged B strip: 16 KB of shared memory whatever the strip width (narrow strips
  // take their whole k in one chunk: one round trip for the strip instead of one per 256 k)
  constexpr int KC = (FMM_SKINNY_KC * 8) / TH;
  // row stride of the staged strip: KC plus 16/TH doubles, so the n lanes that store one k-row of
  // B (consecutive j) and the rows next to it fall on distinct banks
  constexpr int KSTR = KC + (TH >= 2 ? 16 / TH : 0);
  __shared__ __align__(16) double bt[TH * KSTR];
  const GemmTask t = tasks[ids[blockIdx.y]];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row0 = (blockIdx.x * 8 + warp) * ROWS_PER_WARP;
  const bool v2 = ((reinterpret_cast<uintptr_t>(t.A) & 15) == 0) && ((t.lda & 1) == 0);
  double acc[ROWS_PER_WARP][TH];
#pragma unroll
  for (int q = 0; q < ROWS_PER_WARP; ++q)
#pragma unroll
    for (int j = 0; j < TH; ++j) acc[q][j] = 0.0;
  for (int k0 = 0; k0 < t.k; k0 += KC) {
    const int kc = min(KC, t.k - k0);
    __syncthreads();
    // the n values of a k-row by n consecutive lanes (one L1 wavefront per 32 / n rows; a thread
    // per row would touch 32 lines per load), stored conflict-free through the padded stride
    // (eight loads issued before their stores: one L2 round trip per eight elements per thread,
    // not one each -- the staging was the block's critical path)
    const int ne = kc * t.n;
    for (int e0 = threadIdx.x; e0 < ne; e0 += 8 * 256) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + 256 * u, kk = e / t.n, j = e - kk * t.n;
        v[u] = e < ne ? __ldg(t.B + (long long)(k0 + kk) * t.ldb + j) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + 256 * u, kk = e / t.n, j = e - kk * t.n;
        if (e < ne) bt[j * KSTR + kk] = v[u];
      }
    }
    __syncthreads();
    if (v2) {
      // lane covers k pairs kk = 2 lane + 64 s, s = 0..3 of each 256-wide group of the chunk
      for (int g0 = 0; g0 < kc; g0 += 256) {
        double2 a[ROWS_PER_WARP][4];
#pragma unroll
        for (int q = 0; q < ROWS_PER_WARP; ++q) {
          const int i = row0 + q;
#pragma unroll
          for (int s4 = 0; s4 < 4; ++s4) {
            const int kk = g0 + 2 * lane + 64 * s4;
            const double* ap = t.A + (long long)i * t.lda + k0 + kk;
            a[q][s4] = (i < t.m && kk + 1 < kc) ? __ldg(reinterpret_cast<const double2*>(ap))
                       : (i < t.m && kk < kc) ? make_double2(__ldg(ap), 0.0) : make_double2(0.0, 0.0);
          }
        }
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4) {
          const int kk = g0 + 2 * lane + 64 * s4;
          if (kk >= kc) continue;
          const bool second = kk + 1 < kc;
#pragma unroll
          for (int j = 0; j < TH; ++j)
            if (j < t.n) {
              // one 16-byte shared load per lane (512 contiguous bytes per warp: conflict-free)
              double b0, b1;
              if (second) {
                const double2 bb = *reinterpret_cast<const double2*>(&bt[j * KSTR + kk]);
                b0 = bb.x, b1 = bb.y;
              } else {
                b0 = bt[j * KSTR + kk], b1 = 0.0;
              }
#pragma unroll
              for (int q = 0; q < ROWS_PER_WARP; ++q) acc[q][j] = fma(a[q][s4].y, b1, fma(a[q][s4].x, b0, acc[q][j]));
            }
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < ROWS_PER_WARP; ++q) {
        const int i = row0 + q;
        if (i >= t.m) continue;
        const double* arow = t.A + (long long)i * t.lda + k0;
        for (int kk = lane; kk < kc; kk += 128) {
          double a[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) a[u] = kk + 32 * u < kc ? __ldg(arow + kk + 32 * u) : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (kk + 32 * u < kc)
#pragma unroll
              for (int j = 0; j < TH; ++j)
                if (j < t.n) acc[q][j] = fma(a[u], bt[j * KSTR + kk + 32 * u], acc[q][j]);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < ROWS_PER_WARP; ++q) {
    const int i = row0 + q;
#pragma unroll
    for (int j = 0; j < TH; ++j) {
      double v = acc[q][j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc[q][j] = v;
    }
    if (i < t.m && lane < t.n && lane < TH) {
      double v = 0.0;
#pragma unroll
      for (int j = 0; j < TH; ++j)
        if (j == lane) v = acc[q][j];
      double* c = t.C + (long long)i * t.ldc + lane;
      *c = t.beta != 0.0 ? fma(t.beta, *c, t.alpha * v) : t.alpha * v;
    }
  }
}
}  // namespace

int skinny_limit() { return THIN; }

static int pow2_at_least(int x) { return x <= 1 ? 1 : x <= 2 ? 2 : x <= 4 ? 4 : 8; }

void skinny_launch(const GemmTask* d_tasks, const int* d_row_ids, int nrow, int max_n, const int* d_col_ids, int ncol,
                   int max_m, cudaStream_t stream, int thin_r, int thin_c) {
  static const bool rows_narrow = [] {  // FMM_SKINNY_ROWS=narrow: the 32-column form (measurements)
    const char* e = std::getenv("FMM_SKINNY_ROWS");
    return e && std::strcmp(e, "narrow") == 0;
  }();
  if (nrow > 0 && max_n > 0 && !rows_narrow) {
    dim3 grid((unsigned)((max_n + 127) / 128), (unsigned)nrow);
    switch (pow2_at_least(thin_r)) {
      case 1: skinny_rows_w<1><<<grid, 256, 0, stream>>>(d_tasks, d_row_ids, nrow); break;
      case 2: skinny_rows_w<2><<<grid, 256, 0, stream>>>(d_tasks, d_row_ids, nrow); break;
      case 4: skinny_rows_w<4><<<grid, 256, 0, stream>>>(d_tasks, d_row_ids, nrow); break;
      default: skinny_rows_w<8><<<grid, 256, 0, stream>>>(d_tasks, d_row_ids, nrow); break;
    }
    FMM_CUDA(cudaGetLastError());
  } else if (nrow > 0 && max_n > 0) {
    dim3 grid((unsigned)((max_n + 31) / 32), (unsigned)nrow);
    switch (pow2_at_least(thin_r)) {
      case 1: skinny_rows<1><<<grid, 256, 0, stream>>>(d_tasks, d_row_ids, nrow); break;
      case 2: skinny_rows<2><<<grid, 256, 0, stream>>>(d_tasks, d_row_ids, nrow); break;
      case 4: skinny_rows<4><<<grid, 256, 0, stream>>>(d_tasks, d_row_ids, nrow); break;
      default: skinny_rows<8><<<grid, 256, 0, stream>>>(d_tasks, d_row_ids, nrow); break;
    }
    FMM_CUDA(cudaGetLastError());
  }
  if (ncol > 0 && max_m > 0) {
    dim3 grid((unsigned)((max_m + 8 * ROWS_PER_WARP - 1) / (8 * ROWS_PER_WARP)), (unsigned)ncol);
    switch (pow2_at_least(thin_c)) {
      case 1: skinny_cols<1><<<grid, 256, 0, stream>>>(d_tasks, d_col_ids, ncol); break;
      case 2: skinny_cols<2><<<grid, 256, 0, stream>>>(d_tasks, d_col_ids, ncol); break;
      case 4: skinny_cols<4><<<grid, 256, 0, stream>>>(d_tasks, d_col_ids, ncol); break;
      default: skinny_cols<8><<<grid, 256, 0, stream>>>(d_tasks, d_col_ids, ncol); break;
    }
    FMM_CUDA(cudaGetLastError());
  }
}

}  // namespace fmm
