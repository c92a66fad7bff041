// One-launch path for small one-level problems (option small_fused).
//
// Below the paper's cutoff rule (Sec. 3.4: a recursive step pays only when the
// sub-problems sit on the flat part of the dgemm curve) a one-level plan is launch bound: its R
// leaf products give the leaf GEMM's 128-row tiles too few CTAs to fill 148 SMs (c1, Strassen
// 256^3: 7 CTAs), and four dependent launches (formation of S_r, of T_r, the products, the
// assembly) cost more than the arithmetic.  Here the
// whole step C = A * B with one recursion level is ONE launch.  CTA (pos, r) owns a
// 32 x 32 tile `pos` of the leaf grid and product r:
//   1. stages, chunk by chunk along k, the sub-tiles of the A blocks with u_ir != 0 (rows of its
//      tile) and of the B blocks with v_jr != 0 (columns of its tile) in shared memory with
//      cp.async, the next chunk's copies in flight while the current chunk is multiplied;
//   2. forms the chunk of S_r = sum_i u_ir A_i and T_r = sum_j v_jr B_j (Eq. lowrank)
//      from those sub-tiles in shared memory (the sums in the table's block order, first term
//      initialised, no FMA contraction: the values of the separate formation kernels without
//      CSE) and multiplies it on the FP64 tensor pipe (mma.sync.m8n8k4.f64 = DMMA): 16 warps,
//      four groups of four 16 x 16 warp tiles, group g taking the k-steps = g mod 4; the groups'
//      partial tiles are added in group order into M_r's tile;
//   3. writes the tile to a scratch buffer, and the last of the R CTAs of `pos` to finish (a
//      device counter, threadfence-reduction pattern) forms every output block's tile
//      C_k = sum_r w_kr M_r in ascending r, first term initialised -- so the result
//      does not depend on which CTA finishes last -- and resets the counter for the next launch.
// Tiles, chunks and the operand grids are bounds-checked: ragged leaf shapes are zero filled.
// The assembly stages the R product tiles in shared memory (all copies in flight at once) and
// reads them from there.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include "fmm_internal.h"

namespace fmm {

namespace {
constexpr int TM = 32, TN = 32, THREADS = 512;  // 16 warps: 4 groups of 4 (a 16 x 16 sub-tile each)
constexpr int SMEM_BUDGET = 200 * 1024;  // dynamic shared memory of the launch (opt-in)

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
// a copy of `bytes` (0, 8 or 16) bytes, zero-filled to its full size (8, or 16 when vec2)
__device__ __forceinline__ void cpn(unsigned dst, const double* src, unsigned bytes, int vec2) {
  if (vec2)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(bytes ? src : nullptr), "r"(bytes)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(bytes ? src : nullptr), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp16(unsigned dst, const double* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

// CL: the R CTAs of a tile form a thread-block cluster (R <= 16); each keeps its M_r tile in
// shared memory and CTA k < MN forms C_k's tile from its peers' tiles over distributed shared
// memory (no scratch round trip, no counter).  Otherwise the last CTA of the tile does it.
template <bool CL>
__global__ void __launch_bounds__(THREADS) small_fmm_kernel(SmallArgs a) {
  extern __shared__ double smem[];
  __shared__ SmallTerm tu[64], tv[64], tw[256];
  __shared__ int wo[65];
  __shared__ int is_last;
  __shared__ __align__(16) double mts[CL ? TM * TN : 2];
  const int npos = a.tiles_m * a.tiles_n;
  const int pos = CL ? blockIdx.x / a.R : blockIdx.x % npos, r = CL ? blockIdx.x % a.R : blockIdx.x / npos;
  const int i0 = (pos / a.tiles_n) * TM, j0 = (pos % a.tiles_n) * TN;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int grp = warp >> 2, sub = warp & 3;  // group grp takes the k-steps ks = grp mod 4
  const int wm = (sub >> 1) * 16, wn = (sub & 1) * 16;
  const int u0 = __ldg(&a.u_off[r]), nu = __ldg(&a.u_off[r + 1]) - u0;
  const int v0 = __ldg(&a.v_off[r]), nv = __ldg(&a.v_off[r + 1]) - v0;
  if (t < nu) tu[t] = a.u_terms[u0 + t];
  if (t < nv) tv[t] = a.v_terms[v0 + t];
  __syncthreads();
  const int KC = a.kc, LDA = KC + 4, LDB = TN + 8;
  const int stage = nu * TM * LDA + nv * KC * LDB;  // doubles per raw chunk buffer
  double* sS = smem + 2 * a.stage_max;              // formed S_r chunk: TM x LDA
  double* sT = sS + TM * LDA;                       // formed T_r chunk: KC x LDB
  // stage chunk k0 of every term's sub-tile into raw buffer b.  KC is a power of two and each
  // thread keeps one column (pair) of the chunk, stepping down the rows: no division in the loop.
  // 16-byte copies (two columns) where every view is 16-byte aligned (a.vec2), else 8-byte copies;
  // the source size of a copy clips it at the operand's edge (zero fill).
  const int lkc = a.kc_log2;
  const int vw = a.vec2 ? 2 : 1;                           // doubles per copy
  const int lcp = lkc - (a.vec2 ? 1 : 0);                  // log2 of copies per A chunk row
  const int a_col = (t & ((1 << lcp) - 1)) * vw, a_row0 = t >> lcp, a_step = THREADS >> lcp;
  const int b_col = (t & (TN / vw - 1)) * vw, b_row0 = t / (TN / vw), b_step = THREADS / (TN / vw);
  auto load = [&](int k0, int b) {
    const unsigned base = smem_u32(smem + b * a.stage_max);
    const int ka = k0 + a_col;
    const unsigned a_bytes = (unsigned)max(0, min(vw, a.pk - ka)) * 8u;
    for (int q = 0; q < nu; ++q) {
      const double* src = a.A + tu[q].off + (long long)i0 * a.lda + ka;
      const unsigned dst = base + 8u * (unsigned)(q * TM * LDA + a_col);
      for (int i = a_row0; i < TM; i += a_step) {
        const unsigned nb = i0 + i < a.pm ? a_bytes : 0u;
        cpn(dst + 8u * (unsigned)(i * LDA), src + (long long)i * a.lda, nb, a.vec2);
      }
    }
    const int jb = j0 + b_col;
    const unsigned b_bytes = (unsigned)max(0, min(vw, a.pn - jb)) * 8u;
    for (int q = 0; q < nv; ++q) {
      const double* src = a.B + tv[q].off + (long long)k0 * a.ldb + jb;
      const unsigned dst = base + 8u * (unsigned)(nu * TM * LDA + q * KC * LDB + b_col);
      for (int kk = b_row0; kk < KC; kk += b_step) {
        const unsigned nb = k0 + kk < a.pk ? b_bytes : 0u;
        cpn(dst + 8u * (unsigned)(kk * LDB), src + (long long)kk * a.ldb, nb, a.vec2);
      }
    }
    cp_commit();
  };
  (void)stage;
  double acc[2][2][2] = {};
  const int nchunks = (a.pk + KC - 1) / KC;
  load(0, 0);
  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) {
      load((c + 1) * KC, (c + 1) & 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    // form the chunk of S_r and T_r from the staged sub-tiles (independent elements: the loads of
    // several elements are in flight at once)
    const double* ra = smem + (c & 1) * a.stage_max;
    const double* rb = ra + nu * TM * LDA;
    {
      const int col = t & (KC - 1);
      for (int i = t >> lkc; i < TM; i += THREADS >> lkc) {
        const int off = i * LDA + col;
        double v = nu ? __dmul_rn(tu[0].coef, ra[off]) : 0.0;
        for (int q = 1; q < nu; ++q) v = __dadd_rn(v, __dmul_rn(tu[q].coef, ra[q * TM * LDA + off]));
        sS[off] = v;
      }
      const int j = t & (TN - 1);
      for (int kk = t / TN; kk < KC; kk += THREADS / TN) {
        const int off = kk * LDB + j;
        double v = nv ? __dmul_rn(tv[0].coef, rb[off]) : 0.0;
        for (int q = 1; q < nv; ++q) v = __dadd_rn(v, __dmul_rn(tv[q].coef, rb[q * KC * LDB + off]));
        sT[off] = v;
      }
    }
    __syncthreads();
    const int ksteps = (min(KC, a.pk - c * KC) + 3) / 4;
#pragma unroll 2
    for (int ks = grp; ks < ksteps; ks += 4) {
      double fa[2], fb[2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) fa[mi] = sS[(wm + mi * 8 + (lane >> 2)) * LDA + ks * 4 + (lane & 3)];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) fb[ni] = sT[(ks * 4 + (lane & 3)) * LDB + wn + ni * 8 + (lane >> 2)];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni], fa[mi], fb[ni]);
    }
    __syncthreads();  // the raw buffer (c & 1) and the formed chunk are overwritten next
  }
  // the four groups' partial sums, added in group order (deterministic), then M_r's tile ->
  // scratch (tile-major: [r][pos][TM][TN])
  double* red = smem;  // 3 x TM x TN doubles (the raw buffers are free now)
  if (grp > 0) {
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
        *reinterpret_cast<double2*>(red + (grp - 1) * TM * TN + (wm + mi * 8 + (lane >> 2)) * TN + wn + ni * 8 +
                                    2 * (lane & 3)) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
  }
  __syncthreads();
  if (grp == 0) {
    double* mt = CL ? mts : a.Mbuf + ((long long)r * npos + pos) * (TM * TN);
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) {
        const int o = (wm + mi * 8 + (lane >> 2)) * TN + wn + ni * 8 + 2 * (lane & 3);
        double2 v = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
#pragma unroll
        for (int g = 0; g < 3; ++g) {
          const double2 p = *reinterpret_cast<const double2*>(red + g * TM * TN + o);
          v.x = __dadd_rn(v.x, p.x);
          v.y = __dadd_rn(v.y, p.y);
        }
        *reinterpret_cast<double2*>(mt + o) = v;
      }
  }
  if constexpr (CL) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int MN = a.M * a.N;
    if (r < MN) {
      for (int q = t; q <= MN; q += THREADS) wo[q] = __ldg(&a.w_off[q]);
      for (int q = t; q < a.nw; q += THREADS) tw[q] = a.w_terms[q];
    }
    cluster.sync();  // every M_r tile of this position is in its CTA's shared memory
    if (r < MN) {
      const int w0 = wo[r], w1 = wo[r + 1];
      const int kr = r / a.N, kc = r % a.N;
      double* crow = a.C + (long long)(kr * a.pm + i0) * a.ldc + (long long)kc * a.pn + j0;
      for (int e = t; e < TM * TN; e += THREADS) {
        const int i = e >> 5, j = e & 31;
        double s = 0.0;
        for (int q = w0; q < w1; ++q) {
          const double* peer = cluster.map_shared_rank(mts, tw[q].blk);
          const double x = __dmul_rn(tw[q].coef, peer[e]);
          s = q == w0 ? x : __dadd_rn(s, x);
        }
        if (i0 + i < a.pm && j0 + j < a.pn) crow[(long long)i * a.ldc + j] = s;
      }
    }
    cluster.sync();  // the peers' tiles stay until every reader is done
    return;
  }
  __threadfence();
  __syncthreads();
  if (t == 0) is_last = atomicAdd(&a.cnt[pos], 1u) == (unsigned)(a.R - 1);
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // the last CTA of this tile: stage the R product tiles (G positions at a time, every copy in
  // flight at once) and the W terms, then C_k tile = sum_r w_kr M_r tile for every output block k
  const int MN = a.M * a.N, G = a.g;
  for (int k = t; k <= MN; k += THREADS) wo[k] = __ldg(&a.w_off[k]);
  for (int q = t; q < a.nw; q += THREADS) tw[q] = a.w_terms[q];
  const unsigned sbase = smem_u32(smem);
  for (int p0 = 0; p0 < TM * TN; p0 += G) {
    for (int e = t; e < a.R * (G / 2); e += THREADS) {
      const int q = e / (G / 2), h = e % (G / 2);
      cp16(sbase + 8u * (unsigned)(q * G + 2 * h), a.Mbuf + ((long long)q * npos + pos) * (TM * TN) + p0 + 2 * h);
    }
    cp_commit();
    cp_wait<0>();
    __syncthreads();
    for (int k = 0; k < MN; ++k) {
      const int w0 = wo[k], w1 = wo[k + 1];
      const int kr = k / a.N, kc = k % a.N;
      double* crow = a.C + (long long)(kr * a.pm + i0) * a.ldc + (long long)kc * a.pn + j0;
      for (int e = t; e < G; e += THREADS) {
        const int i = (p0 + e) >> 5, j = (p0 + e) & 31;
        double s = 0.0;
        for (int q = w0; q < w1; ++q) {
          const double x = __dmul_rn(tw[q].coef, smem[tw[q].blk * G + e]);
          s = q == w0 ? x : __dadd_rn(s, x);
        }
        if (i0 + i < a.pm && j0 + j < a.pn) crow[(long long)i * a.ldc + j] = s;
      }
    }
    __syncthreads();
  }
  if (t == 0) a.cnt[pos] = 0u;  // ready for the next launch (stream ordered)
}
}  // namespace

int small_tile() { return TM; }

// chunk depth and assembly group of a launch: the largest k-chunk (a power of two from 4, at most
// the leaf depth rounded up) whose two staging buffers fit the budget; the largest group of positions
// (a power of two, 256 .. 1024) whose R product values fit
bool small_config(int max_nu, int max_nv, int pk, int R, int* kc, int* g) {
  int k = 4;
  while (k < pk && k < 256) k *= 2;
  // two raw buffers and the formed chunk of S_r and T_r
  auto bytes = [&](int kk) { return 8 * ((2 * max_nu + 1) * TM * (kk + 4) + (2 * max_nv + 1) * kk * (TN + 8)); };
  while (k > 4 && bytes(k) > SMEM_BUDGET) k /= 2;
  if (bytes(k) > SMEM_BUDGET || max_nu > 64 || max_nv > 64) return false;
  int gg = 1024;
  while (gg > 256 && 8 * R * gg > SMEM_BUDGET) gg /= 2;
  if (8 * R * gg > SMEM_BUDGET) return false;
  *kc = k;
  *g = gg;
  return true;
}

// whether the cluster variant can run a launch of R-CTA clusters (R <= 16, at least one cluster
// co-resident with this dynamic shared memory)
bool small_cluster_ok(int R, int smem) {
  if (R > 16 || R < 1) return false;
  static std::atomic<unsigned long long> configured{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    FMM_CUDA(cudaFuncSetAttribute(small_fmm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BUDGET));
    FMM_CUDA(cudaFuncSetAttribute(small_fmm_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured.fetch_or(bit);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)R);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = (size_t)smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)R;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, small_fmm_kernel<true>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return n > 0;
}

void small_launch(const SmallArgs& a, cudaStream_t stream) {
  const long long grid = (long long)a.tiles_m * a.tiles_n * a.R;
  if (grid <= 0) return;
  if (a.cluster) {  // attributes were set by small_cluster_ok at plan time
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = (size_t)a.smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)a.R;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    FMM_CUDA(cudaLaunchKernelEx(&cfg, small_fmm_kernel<true>, a));
    return;
  }
  static std::atomic<unsigned long long> configured{0};
  int dev = 0;
  FMM_CUDA(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    FMM_CUDA(cudaFuncSetAttribute(small_fmm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BUDGET));
    configured.fetch_or(bit);
  }
  small_fmm_kernel<false><<<(unsigned)grid, THREADS, (size_t)a.smem, stream>>>(a);
  FMM_CUDA(cudaGetLastError());
}

}  // namespace fmm
