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
#include <cstdlib>

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
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// CL: the R CTAs of a tile form a thread-block cluster (R <= 16); each keeps its M_r tile in
// shared memory and CTA k < MN forms C_k's tile from its peers' tiles over distributed shared
// memory (no scratch round trip, no counter).  Otherwise the last CTA of the tile does it.
#ifdef FMM_SMALL_TIMING  // diagnostics build: phase timestamps (globaltimer, ns) of CTA 0 and of the
                         // last CTA of tile 0, printed by thread 0
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}
#define TSTAMP(i) (tst[i] = gtime())
#else
#define TSTAMP(i) ((void)0)
#endif
template <bool CL, int KC, int V>
__global__ void __launch_bounds__(THREADS) small_fmm_kernel(SmallArgs a) {
#ifdef FMM_SMALL_TIMING
  unsigned long long tst[10] = {};
#endif
  TSTAMP(0);
  extern __shared__ double smem[];
  __shared__ SmallTerm tu[64], tv[64], tw[256];
  __shared__ int wo[65];
  __shared__ int is_last;
  __shared__ __align__(16) double mts[CL ? TM * TN : 2];
  constexpr int LDA = KC + 4, LDB = TN + 8;        // raw / formed chunk row strides (doubles)
  constexpr int ACP = KC / V, BCP = TN / V;        // copies per A / B chunk row
  constexpr int ACT = (TM * ACP + THREADS - 1) / THREADS, BCT = (KC * BCP + THREADS - 1) / THREADS;
  constexpr int SPT = (TM * KC + THREADS - 1) / THREADS, TPT = (KC * TN + THREADS - 1) / THREADS;
  const int npos = a.tiles_m * a.tiles_n;
  const int pos = CL ? blockIdx.x / a.R : blockIdx.x % npos, r = CL ? blockIdx.x % a.R : blockIdx.x / npos;
  const int i0 = (pos / a.tiles_n) * TM, j0 = (pos % a.tiles_n) * TN;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int grp = warp >> 2, sub = warp & 3;  // group grp takes the k-steps ks = grp mod 4
  const int wm = (sub >> 1) * 16, wn = (sub & 1) * 16;
  const int u0 = a.u_off[r], nu = a.u_off[r + 1] - u0;
  const int v0 = a.v_off[r], nv = a.v_off[r + 1] - v0;
  if (t < nu) tu[t] = a.u_terms[u0 + t];
  if (t < nv) tv[t] = a.v_terms[v0 + t];
  const int MN = a.M * a.N;
  __syncthreads();
  TSTAMP(1);
  const int stage = a.stage_max;            // doubles per raw chunk buffer
  double* sS = smem + 2 * stage;            // formed S_r chunk: TM x LDA
  double* sT = sS + TM * LDA;               // formed T_r chunk: KC x LDB
  // stage chunk k0 of every term's sub-tile into raw buffer b: every index below is a compile-time
  // shift of the thread id; the source size of a copy clips it at the operand's edge (zero fill)
  auto load = [&](int k0, int b) {
    const unsigned base = smem_u32(smem + b * stage);
#pragma unroll
    for (int it = 0; it < ACT; ++it) {
      const int e = t + it * THREADS, i = e / ACP, col = (e % ACP) * V;
      if (e < TM * ACP) {
        const unsigned nb = i0 + i < a.pm ? (unsigned)max(0, min(V, a.pk - k0 - col)) * 8u : 0u;
        const long long go = (long long)(i0 + i) * a.lda + k0 + col;
        const unsigned so = 8u * (unsigned)(i * LDA + col);
        for (int q = 0; q < nu; ++q) cpn(base + 8u * (unsigned)(q * TM * LDA) + so, a.A + tu[q].off + go, nb, V == 2);
      }
    }
    const unsigned bb = base + 8u * (unsigned)(nu * TM * LDA);
#pragma unroll
    for (int it = 0; it < BCT; ++it) {
      const int e = t + it * THREADS, kk = e / BCP, col = (e % BCP) * V;
      if (e < KC * BCP) {
        const unsigned nb = k0 + kk < a.pk ? (unsigned)max(0, min(V, a.pn - j0 - col)) * 8u : 0u;
        const long long go = (long long)(k0 + kk) * a.ldb + j0 + col;
        const unsigned so = 8u * (unsigned)(kk * LDB + col);
        for (int q = 0; q < nv; ++q) cpn(bb + 8u * (unsigned)(q * KC * LDB) + so, a.B + tv[q].off + go, nb, V == 2);
      }
    }
    cp_commit();
  };
  double acc[2][2][2] = {};
  const int nchunks = (a.pk + KC - 1) / KC;
  load(0, 0);
  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks && a.prefetch) {
      load((c + 1) * KC, (c + 1) & 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (c == 0) TSTAMP(2);
    // form the chunk of S_r and T_r from the staged sub-tiles: terms outside, the thread's
    // elements (independent) inside, so their shared-memory loads are in flight together
    const double* ra = smem + (c & 1) * stage;
    const double* rb = ra + nu * TM * LDA;
    {
      double vs[SPT], vt[TPT];
#pragma unroll
      for (int it = 0; it < SPT; ++it) vs[it] = 0.0;
#pragma unroll
      for (int it = 0; it < TPT; ++it) vt[it] = 0.0;
      for (int q = 0; q < nu; ++q) {
        const double cf = tu[q].coef;
#pragma unroll
        for (int it = 0; it < SPT; ++it) {
          const int e = t + it * THREADS;
          const double x = __dmul_rn(cf, ra[q * TM * LDA + (e / KC) * LDA + e % KC]);
          vs[it] = q == 0 ? x : __dadd_rn(vs[it], x);
        }
      }
      for (int q = 0; q < nv; ++q) {
        const double cf = tv[q].coef;
#pragma unroll
        for (int it = 0; it < TPT; ++it) {
          const int e = t + it * THREADS;
          const double x = __dmul_rn(cf, rb[q * KC * LDB + (e / TN) * LDB + e % TN]);
          vt[it] = q == 0 ? x : __dadd_rn(vt[it], x);
        }
      }
#pragma unroll
      for (int it = 0; it < SPT; ++it) {
        const int e = t + it * THREADS;
        if (e < TM * KC) sS[(e / KC) * LDA + e % KC] = vs[it];
      }
#pragma unroll
      for (int it = 0; it < TPT; ++it) {
        const int e = t + it * THREADS;
        if (e < KC * TN) sT[(e / TN) * LDB + e % TN] = vt[it];
      }
    }
    __syncthreads();
#pragma unroll
    for (int ks = grp; ks < KC / 4; ks += 4) {  // zero-filled k beyond the leaf depth adds zeros
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
    if (c == 0) TSTAMP(3);
    if (!a.prefetch && c + 1 < nchunks) load((c + 1) * KC, (c + 1) & 1);
  }
  TSTAMP(4);
  // the W terms (any CTA may assemble), read while the product tile is stored
  for (int q = t; q <= MN; q += THREADS) wo[q] = a.w_off[q];
  for (int q = t; q < a.nw; q += THREADS) tw[q] = a.w_terms[q];
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
  if (a.direct) {  // L = 0: the tile is C's (w = 1); no assembly
    if (grp == 0) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          const int row = wm + mi * 8 + (lane >> 2), col = wn + ni * 8 + 2 * (lane & 3);
          const int o = row * TN + col;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double v = acc[mi][ni][h];
#pragma unroll
            for (int g = 0; g < 3; ++g) v = __dadd_rn(v, red[g * TM * TN + o + h]);
            if (i0 + row < a.pm && j0 + col + h < a.pn) a.C[(long long)(i0 + row) * a.ldc + j0 + col + h] = v;
          }
        }
    }
    return;
  }
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
  if (a.coop) {
    // every CTA of the grid is resident (checked by the host): the R CTAs of this tile wait for
    // each other (counter `arrive`), then each forms C_k for its own slice of the tile's rows from
    // all R product tiles (staged in shared memory), and the last to leave (`depart`) resets both
    // counters for the next launch
    unsigned* arrive = a.cnt + pos;
    unsigned* depart = a.cnt + npos + pos;
    if (t == 0) {
      atomicAdd(arrive, 1u);
      while (ld_acquire_u32(arrive) < (unsigned)a.R) __nanosleep(32);
    }
    __syncthreads();
    TSTAMP(5);
    const int rlo = r * TM / a.R, rhi = (r + 1) * TM / a.R, P = (rhi - rlo) * TN;
    if (P > 0) {
      const unsigned sbase = smem_u32(smem);
      for (int e = t; e < a.R * (P / 2); e += THREADS) {
        const int q = e / (P / 2), h = e % (P / 2);
        cp16(sbase + 8u * (unsigned)(q * P + 2 * h), a.Mbuf + ((long long)q * npos + pos) * (TM * TN) + rlo * TN + 2 * h);
      }
      cp_commit();
      cp_wait<0>();
      __syncthreads();
      TSTAMP(6);
      for (int x = t; x < P * MN; x += THREADS) {  // one (output block, position) per thread
        const int k = x / P, e = x % P;
        const int i = rlo + e / TN, j = e % TN;
        if (i0 + i >= a.pm || j0 + j >= a.pn) continue;
        const int w0 = wo[k], w1 = wo[k + 1];
        double s = 0.0;
        for (int q = w0; q < w1; ++q) {
          const double v = __dmul_rn(tw[q].coef, smem[tw[q].blk * P + e]);
          s = q == w0 ? v : __dadd_rn(s, v);
        }
        a.C[(long long)((k / a.N) * a.pm + i0 + i) * a.ldc + (long long)(k % a.N) * a.pn + j0 + j] = s;
      }
    }
    __syncthreads();
    if (t == 0 && atomicAdd(depart, 1u) == (unsigned)(a.R - 1)) {
      *arrive = 0u;
      *depart = 0u;
    }
#ifdef FMM_SMALL_TIMING
    if (pos == 0 && r == 0 && t == 0)
      printf("small coop cta0: start %llu prologue %llu chunk0-ready %llu loop-done %llu arrived %llu staged %llu end %llu\n",
             tst[0] % 1000000000ull, tst[1] - tst[0], tst[2] - tst[0], tst[4] - tst[0], tst[5] - tst[0], tst[6] - tst[0],
             gtime() - tst[0]);
#endif
    return;
  }
  if (t == 0) is_last = atomicAdd(&a.cnt[pos], 1u) == (unsigned)(a.R - 1);
  __syncthreads();
  TSTAMP(5);
#ifdef FMM_SMALL_TIMING
  if (blockIdx.x == 0 && t == 0)
    printf("small cta0: start %llu prologue %llu chunk0-ready %llu chunk0-done %llu loop-done %llu counted %llu\n",
           tst[0] % 1000000000ull, tst[1] - tst[0], tst[2] - tst[0], tst[3] - tst[0], tst[4] - tst[0], tst[5] - tst[0]);
#endif
  if (!is_last) return;
  __threadfence();
  // the last CTA of this tile: stage the R product tiles (G positions at a time, every copy in
  // flight at once) and the W terms, then C_k tile = sum_r w_kr M_r tile for every output block k
  const int G = a.g;
  const unsigned sbase = smem_u32(smem);
  for (int p0 = 0; p0 < TM * TN; p0 += G) {
    for (int e = t; e < a.R * (G / 2); e += THREADS) {
      const int q = e / (G / 2), h = e % (G / 2);
      cp16(sbase + 8u * (unsigned)(q * G + 2 * h), a.Mbuf + ((long long)q * npos + pos) * (TM * TN) + p0 + 2 * h);
    }
    cp_commit();
    cp_wait<0>();
    __syncthreads();
    if (p0 == 0) TSTAMP(6);
    // each thread's positions of the group side by side (independent chains), terms in r order
    constexpr int PPT = TM * TN / THREADS;
    for (int k = 0; k < MN; ++k) {
      const int w0 = wo[k], w1 = wo[k + 1];
      const int kr = k / a.N, kc = k % a.N;
      double* crow = a.C + (long long)(kr * a.pm + i0) * a.ldc + (long long)kc * a.pn + j0;
      double sacc[PPT];
#pragma unroll
      for (int p = 0; p < PPT; ++p) sacc[p] = 0.0;
      for (int q = w0; q < w1; ++q) {
        const double cf = tw[q].coef;
        const double* mq = smem + tw[q].blk * G;
#pragma unroll
        for (int p = 0; p < PPT; ++p) {
          const int e = t + p * THREADS;
          if (e < G) {
            const double x = __dmul_rn(cf, mq[e]);
            sacc[p] = q == w0 ? x : __dadd_rn(sacc[p], x);
          }
        }
      }
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        const int e = t + p * THREADS;
        const int i = (p0 + e) >> 5, j = (p0 + e) & 31;
        if (e < G && i0 + i < a.pm && j0 + j < a.pn) crow[(long long)i * a.ldc + j] = sacc[p];
      }
    }
    __syncthreads();
  }
  if (t == 0) a.cnt[pos] = 0u;  // ready for the next launch (stream ordered)
#ifdef FMM_SMALL_TIMING
  if (pos == 0 && t == 0)
    printf("small last of tile 0 (r %d): start %llu prologue %llu chunk0-ready %llu loop-done %llu counted %llu "
           "staged %llu end %llu\n", r, tst[0] % 1000000000ull, tst[1] - tst[0], tst[2] - tst[0], tst[4] - tst[0],
           tst[5] - tst[0], tst[6] - tst[0], gtime() - tst[0]);
#endif
}
}  // namespace

int small_tile() { return TM; }

// chunk depth and assembly group of a launch: the k-chunk (16, 32 or 64: the leaf depth rounded
// up, at most 64) whose two staging buffers fit the budget; the largest group of positions
// (a power of two, 256 .. 1024) whose R product values fit
bool small_config(int max_nu, int max_nv, int pk, int R, int* kc, int* g) {
  // two raw buffers and the formed chunk of S_r and T_r
  auto bytes = [&](int kk) { return 8 * ((2 * max_nu + 1) * TM * (kk + 4) + (2 * max_nv + 1) * kk * (TN + 8)); };
  int k = pk <= 16 ? 16 : pk <= 32 ? 32 : 64;
  if (const char* e = getenv("FMM_SMALL_KC")) k = std::min(k, std::max(16, atoi(e)));  // diagnostics
  while (k > 16 && bytes(k) > SMEM_BUDGET) k /= 2;
  if (bytes(k) > SMEM_BUDGET || max_nu > 64 || max_nv > 64) return false;
  int gg = 1024;
  while (gg > 256 && 8 * R * gg > SMEM_BUDGET) gg /= 2;
  if (8 * R * gg > SMEM_BUDGET) return false;
  *kc = k;
  *g = gg;
  return true;
}

template <bool CL, int KC, int V>
static void set_attrs() {
  FMM_CUDA(cudaFuncSetAttribute(small_fmm_kernel<CL, KC, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BUDGET));
  if (CL) FMM_CUDA(cudaFuncSetAttribute(small_fmm_kernel<CL, KC, V>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}
static void configure_all() {
  static std::atomic<unsigned long long> configured{0};
  int dev = 0;
  FMM_CUDA(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  if (configured.load() & bit) return;
  set_attrs<false, 16, 1>(), set_attrs<false, 16, 2>(), set_attrs<false, 32, 1>(), set_attrs<false, 32, 2>();
  set_attrs<false, 64, 1>(), set_attrs<false, 64, 2>();
  set_attrs<true, 16, 1>(), set_attrs<true, 16, 2>(), set_attrs<true, 32, 1>(), set_attrs<true, 32, 2>();
  set_attrs<true, 64, 1>(), set_attrs<true, 64, 2>();
  configured.fetch_or(bit);
}
template <bool CL>
static auto kernel_for(int kc, int v) -> void (*)(SmallArgs) {
  if (kc == 16) return v == 2 ? small_fmm_kernel<CL, 16, 2> : small_fmm_kernel<CL, 16, 1>;
  if (kc == 32) return v == 2 ? small_fmm_kernel<CL, 32, 2> : small_fmm_kernel<CL, 32, 1>;
  return v == 2 ? small_fmm_kernel<CL, 64, 2> : small_fmm_kernel<CL, 64, 1>;
}

// whether the cluster variant can run a launch of R-CTA clusters (R <= 16, at least one cluster
// co-resident with this dynamic shared memory)
bool small_cluster_ok(int R, int smem) {
  if (R > 16 || R < 1) return false;
  configure_all();
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
  if (cudaOccupancyMaxActiveClusters(&n, small_fmm_kernel<true, 64, 1>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return n > 0;
}

// whether every CTA of a launch of `grid` CTAs with this dynamic shared memory is co-resident
// (the cooperative assembly waits for the other CTAs of a tile)
bool small_coop_ok(long long grid, int smem, int kc, int vec2) {
  configure_all();
  int per_sm = 0, sms = 0, dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel_for<false>(kc, vec2 ? 2 : 1), THREADS, (size_t)smem) !=
          cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return grid <= (long long)per_sm * sms;
}

void small_launch(const SmallArgs& a, cudaStream_t stream) {
  const long long grid = (long long)a.tiles_m * a.tiles_n * a.R;
  if (grid <= 0) return;
  configure_all();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = (size_t)a.smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  if (a.cluster) {
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)a.R;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
  } else {  // the cooperative assembly's CTAs wait for each other: a cooperative launch guarantees
            // that they are all resident (it fails instead of hanging if they cannot be)
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = (a.cluster || a.coop) ? 1 : 0;
  const int v = a.vec2 ? 2 : 1;
  FMM_CUDA(cudaLaunchKernelEx(&cfg, a.cluster ? kernel_for<true>(a.kc, v) : kernel_for<false>(a.kc, v), a));
}

}  // namespace fmm
