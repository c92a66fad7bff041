// K2 (main path): persistent, warp-specialised grouped FP64 GEMM fed by TMA.
//
// Same contract as grouped_dgemm in fmm_gemm.cu (task table of C = alpha A B + beta C, row-major),
// used whenever every operand view is 16-byte aligned with even leading dimensions (what TMA
// requires).  Structure, per CTA (one per SM, looping over tiles):
//   warpgroup 0 (producer): one thread issues cp.async.bulk.tensor (TMA) loads of the A tile
//       (one 128x16 box) and the B tile (eight 16x16 boxes) per k-step into a 6-stage ring of
//       shared-memory buffers as soon as a stage is released, signalling a "full" mbarrier with
//       complete_tx; it runs over the CTA's whole (tile, k-step) sequence, so the next tile's
//       loads are in flight while the current tile's epilogue runs.  It gives its registers
//       away with setmaxnreg.dec (40), so the consumers can grow to 232 (setmaxnreg.inc) —
//       the 64x32 warp tile needs ~210, above the 168 a flat 384-thread launch would allow.
//   warpgroups 1-2 (consumers): 2 x 4 warps of 64 x 32 outputs; wait "full", read register fragments,
//       issue mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), arrive "empty"; epilogue straight from
//       registers with 16-byte stores.  No CTA-wide barrier in the main loop.
// TMA writes the tiles with the 128-byte swizzle (16-byte chunk index XOR row mod 8).  The DMMA
// fragment pattern (lane -> row lane/4, col lane%4 for A; row lane%4, col lane/4 for B) would hit
// 2- or 4-way bank conflicts on that layout, so fragment rows and columns are mapped to tile rows
// and columns by fixed permutations chosen to make every 8-byte fragment load conflict-free:
//   A: fragment row r of m-subtile i  -> tile row 16*(i/2) + 2r + (i%2)
//   B: fragment col j of n-subtile jj -> tile col 16*(jj/2) + 4*(jj%2) + {0,1,8,9,2,3,10,11}[j]
// The epilogue writes each accumulator to the tile position its operands came from.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "fmm_internal.h"

namespace fmm {

namespace {
constexpr int BM = 128, BK = 16;
constexpr int STAGES_PLAIN = 6, STAGES_FUSED = 6;
constexpr int CONSUMERS = 8, THREADS = 128 + CONSUMERS * 32;  // warpgroup 0 = producer, 1-2 = consumers
constexpr int ADD_WARPS = THREADS / 32;                        // every warp of an addition CTA
constexpr int FUSED_HDR_BYTES = FUSED_PROG_BYTES + 1024;       // program area + barriers, 1 KB aligned
constexpr int A_BYTES = BM * BK * 8;   // 16 KB
constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
constexpr size_t smem_bytes(int bn, int stages, bool fused) {
  return fused ? 1024 /*align*/ + FUSED_HDR_BYTES +
                     cmax((size_t)stages * (A_BYTES + BK * bn * 8), (size_t)ADD_WARPS * 2 * FUSED_ADD_SEG_BYTES)
               : (size_t)stages * (A_BYTES + BK * bn * 8) + 1024 /*align*/ + 256 /*barriers*/;
}
constexpr int GROUP_M = 8;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(unsigned dst, const CUtensorMap* map, int c0, int c1, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// 1-D bulk copy global -> shared (TMA engine, no registers held while in flight)
__device__ __forceinline__ void bulk_load(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ double lds64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ double2 lds128(unsigned addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
// L2-coherent loads: inputs of assembly jobs were written by other SMs during this kernel
__device__ __forceinline__ double2 ldcg2(const double* p) {
  double2 v;
  asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ double ldcg1(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}

struct TileCoord {
  int task, m0, n0;
};
// Uniform launches (every task has the same tile grid, e.g. all leaves of a level) map a tile to
// its task by division; others binary-search the tile prefix sums in the task table.
struct Uniform {
  int tiles, tiles_m, tiles_n;  // tiles == 0: not uniform
};
template <int BN>
__device__ __forceinline__ TileCoord locate(const GemmTask* __restrict__ tasks, int ntasks, int tile, Uniform u) {
  int lo, tiles_m, tiles_n, local;
  if (u.tiles) {
    lo = tile / u.tiles;
    local = tile - lo * u.tiles;
    tiles_m = u.tiles_m;
    tiles_n = u.tiles_n;
  } else {
    lo = 0;
    int hi = ntasks - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(&tasks[mid].tile_begin) <= tile) lo = mid; else hi = mid - 1;
    }
    tiles_m = __ldg(&tasks[lo].tiles_m);
    tiles_n = __ldg(&tasks[lo].tiles_n);
    local = tile - __ldg(&tasks[lo].tile_begin);
  }
  const int span = GROUP_M * tiles_n;
  const int group = local / span;
  const int first_m = group * GROUP_M;
  const int gsize = min(tiles_m - first_m, GROUP_M);
  const int tm = first_m + (local % span) % gsize;
  const int tn = (local % span) / gsize;
  return {lo, tm * BM, tn * BN};
}

// ---- addition-chain interpreter (fused kernel) -------------------------------------------------
// Chain arithmetic exactly as the generated K1/K3 kernels without CSE and as the oracle: the first
// term initialises (copy / negate / scale), later terms add, subtract or add a product; no FMA.
__device__ __forceinline__ double chain_first(double c, double v) {
  return c == 1.0 ? v : c == -1.0 ? -v : __dmul_rn(c, v);
}
__device__ __forceinline__ double chain_next(double acc, double c, double v) {
  return c == 1.0 ? __dadd_rn(acc, v) : c == -1.0 ? __dsub_rn(acc, v) : __dadd_rn(acc, __dmul_rn(c, v));
}

// A job as one warp sees it: the program (in shared memory) and the node's pointers held in
// registers, lane i owning in[i] / in[32+i] and out[i] / out[32+i] (broadcast with shuffles).
struct JobView {
  const FusedProg* prog;  // shared memory
  const short* ostart;
  const short* tin;
  const double* tcoef;
  unsigned long long pin0, pin1, pout0, pout1;
  long long ld_in, ld_out;
};
__device__ __forceinline__ unsigned long long pick(unsigned long long p0, unsigned long long p1, int idx) {
  return idx < 32 ? __shfl_sync(0xffffffffu, p0, idx) : __shfl_sync(0xffffffffu, p1, idx - 32);
}
__device__ __forceinline__ JobView job_view(const FusedArgs& fa, const char* sprog, const FusedJob& j, int lane) {
  JobView v;
  v.prog = reinterpret_cast<const FusedProg*>(sprog) + j.prog;
  const int nin = v.prog->nin, nout = v.prog->nout;
  v.ostart = reinterpret_cast<const short*>(sprog + v.prog->ostart_off);
  v.tin = reinterpret_cast<const short*>(sprog + v.prog->in_off);
  v.tcoef = reinterpret_cast<const double*>(sprog + v.prog->coef_off);
  const char* nd = fa.base + v.prog->node_off + (long long)j.node * v.prog->node_bytes;
  const unsigned long long* in = reinterpret_cast<const unsigned long long*>(nd);
  const unsigned long long* out = in + nin;
  const long long* lds = reinterpret_cast<const long long*>(out + nout);
  v.pin0 = lane < nin ? __ldg(in + lane) : 0ull;
  v.pin1 = lane + 32 < nin ? __ldg(in + lane + 32) : 0ull;
  v.pout0 = lane < nout ? __ldg(out + lane) : 0ull;
  v.pout1 = lane + 32 < nout ? __ldg(out + lane + 32) : 0ull;
  v.ld_in = __ldg(lds);
  v.ld_out = __ldg(lds + 1);
  return v;
}

// Direct path: every lane loads its columns from global (L2-coherent), U column groups in flight.
// Every loop that contains a shuffle (pointer broadcast) runs the same trip count on all lanes.
template <int U>
__device__ void job_direct(const JobView& v, const FusedJob& j, int lane) {
  const int cols = v.prog->cols, nout = v.prog->nout;
  const bool vec2 = v.prog->vec2 != 0;
  const int step = vec2 ? 64 * U : 32 * U;
  for (int row = j.row0; row < j.row0 + j.nrows; ++row) {
    for (int o = 0; o < nout; ++o) {
      double* y = reinterpret_cast<double*>(pick(v.pout0, v.pout1, o));
      if (!y) continue;
      y += (long long)row * v.ld_out;
      const int t0 = v.ostart[o], t1 = v.ostart[o + 1];
      for (int cb = 0; cb < cols; cb += step) {
        if (vec2) {
          const int c = cb + 2 * lane;
          double2 acc[U];
#pragma unroll
          for (int u = 0; u < U; ++u) acc[u] = make_double2(0.0, 0.0);
          for (int t = t0; t < t1; ++t) {
            const int i = v.tin[t];
            const double coef = v.tcoef[t];
            const double* x = reinterpret_cast<const double*>(pick(v.pin0, v.pin1, i)) + (long long)row * v.ld_in;
            double2 val[U];
#pragma unroll
            for (int u = 0; u < U; ++u) val[u] = c + 64 * u < cols ? ldcg2(x + c + 64 * u) : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < U; ++u) {
              if (t == t0) {
                acc[u].x = chain_first(coef, val[u].x);
                acc[u].y = chain_first(coef, val[u].y);
              } else {
                acc[u].x = chain_next(acc[u].x, coef, val[u].x);
                acc[u].y = chain_next(acc[u].y, coef, val[u].y);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (c + 64 * u < cols) *reinterpret_cast<double2*>(y + c + 64 * u) = acc[u];
        } else {
          const int c = cb + lane;
          double acc[U];
#pragma unroll
          for (int u = 0; u < U; ++u) acc[u] = 0.0;
          for (int t = t0; t < t1; ++t) {
            const int i = v.tin[t];
            const double coef = v.tcoef[t];
            const double* x = reinterpret_cast<const double*>(pick(v.pin0, v.pin1, i)) + (long long)row * v.ld_in;
            double val[U];
#pragma unroll
            for (int u = 0; u < U; ++u) val[u] = c + 32 * u < cols ? ldcg1(x + c + 32 * u) : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u) acc[u] = t == t0 ? chain_first(coef, val[u]) : chain_next(acc[u], coef, val[u]);
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (c + 32 * u < cols) y[c + 32 * u] = acc[u];
        }
      }
    }
  }
}

// Staged path (producer warps 1-3): lane i copies the row segment of input i of a piece into one
// of the warp's two shared-memory buffers with a 1-D bulk copy (TMA engine; nothing held in
// registers); the next piece's copies are in flight while the warp evaluates the chains of the
// current one from shared memory (two column pairs per lane) and stores the outputs (16 bytes).
struct Staging {
  unsigned buf0, bar0;  // buffer b at buf0 + b * FUSED_ADD_SEG_BYTES, its mbarrier at bar0 + 8 b
  unsigned phase;       // bit b = parity of buffer b
};
__device__ void job_staged(const JobView& v, const FusedJob& j, int lane, Staging& st) {
  const int cols = v.prog->cols, nin = v.prog->nin, nout = v.prog->nout, seg = v.prog->seg;
  const int nseg = (cols + seg - 1) / seg;
  const int npieces = j.nrows * nseg;
  auto issue = [&](int p, int b) {
    const int row = j.row0 + p / nseg, c0 = (p % nseg) * seg;
    const int w = min(seg, cols - c0);
    const unsigned bar = st.bar0 + 8u * (unsigned)b;
    if (lane == 0) mbar_expect_tx(bar, (unsigned)(nin * w * 8));
    __syncwarp();
    if (lane < nin)
      bulk_load(st.buf0 + (unsigned)b * FUSED_ADD_SEG_BYTES + (unsigned)(lane * seg * 8),
                reinterpret_cast<const double*>(v.pin0) + (long long)row * v.ld_in + c0, (unsigned)(w * 8), bar);
  };
  if (npieces > 0) issue(0, 0);
  int b = 0;
  for (int p = 0; p < npieces; ++p, b ^= 1) {
    if (p + 1 < npieces) issue(p + 1, b ^ 1);
    mbar_wait(st.bar0 + 8u * (unsigned)b, (st.phase >> b) & 1u);
    st.phase ^= 1u << b;
    const int row = j.row0 + p / nseg, c0 = (p % nseg) * seg;
    const int w = min(seg, cols - c0);
    const unsigned sbuf = st.buf0 + (unsigned)b * FUSED_ADD_SEG_BYTES;
    for (int o = 0; o < nout; ++o) {
      double* y = reinterpret_cast<double*>(pick(v.pout0, v.pout1, o));
      if (!y) continue;
      y += (long long)row * v.ld_out + c0;
      const int t0 = v.ostart[o], t1 = v.ostart[o + 1];
      for (int c = 2 * lane; c < w; c += 128) {
        const bool two = c + 64 < w;
        double2 a0 = make_double2(0.0, 0.0), a1 = a0;
        for (int t = t0; t < t1; ++t) {
          const unsigned xo = sbuf + (unsigned)((v.tin[t] * seg + c) * 8);
          const double coef = v.tcoef[t];
          const double2 x0 = lds128(xo);
          const double2 x1 = two ? lds128(xo + 512u) : make_double2(0.0, 0.0);
          if (t == t0) {
            a0.x = chain_first(coef, x0.x);
            a0.y = chain_first(coef, x0.y);
            a1.x = chain_first(coef, x1.x);
            a1.y = chain_first(coef, x1.y);
          } else {
            a0.x = chain_next(a0.x, coef, x0.x);
            a0.y = chain_next(a0.y, coef, x0.y);
            a1.x = chain_next(a1.x, coef, x1.x);
            a1.y = chain_next(a1.y, coef, x1.y);
          }
        }
        *reinterpret_cast<double2*>(y + c) = a0;
        if (two) *reinterpret_cast<double2*>(y + c + 64) = a1;
      }
    }
    __syncwarp();  // every lane is done with buffer b before it is refilled
  }
}

__device__ __forceinline__ int claim(unsigned long long* ctr, int lane) {
  int idx = 0;
  if (lane == 0) idx = (int)atomicAdd(ctr, 1ull);
  return __shfl_sync(0xffffffffu, idx, 0);
}

// Run one job (formation or assembly) with a whole warp; staged when st != nullptr.
template <int U>
__device__ void run_job(const FusedArgs& fa, const char* sprog, int jidx, int lane, Staging* st) {
  const FusedJob j = fa.jobs[jidx];
  if (j.kind == 1) {  // assembly: wait until every leaf tile of the parent is stored
    if (lane == 0) {
      const unsigned long long target = (unsigned long long)__ldg(&fa.tiles_target[j.dep]);
      while (ld_acquire(&fa.ctr[2 + fa.np + j.dep]) < target) __nanosleep(256);
    }
    __syncwarp();
    fence_proxy_async_global();
  }
  const JobView v = job_view(fa, sprog, j, lane);
  if (st && v.prog->vec2 && v.prog->seg > 0) job_staged(v, j, lane, *st);
  else job_direct<U>(v, j, lane);
  if (j.kind == 0) {  // formation: publish (release) to the TMA readers of the leaf products
    fence_proxy_async_global();
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicAdd(&fa.ctr[2 + j.dep], 1ull);
  }
}

// BN columns per CTA tile, consumer warps arranged WGM x WGN (WGM * WGN = 8); warp tile
// (128 / WGM) x (BN / WGN), both multiples of 16 so the fragment permutations apply.
//
// FUSED: the level-L formation (F) and assembly (A) jobs of the plan run in the same launch,
// spatially partitioned: CTAs [0, gemm_ctas) are GEMM CTAs (one per SM, as the plain kernel),
// CTAs [gemm_ctas, gridDim.x) are addition CTAs whose 12 warps evaluate addition chains with
// bulk-copy staging.  The two must not share an SM: on B200 the FP64 tensor path (DMMA) and the
// FP64 ALU (DADD / DMUL) are one pipe, and a worker warp next to eight DMMA warps was measured to
// get ~1 % of it.  Every warp of the GPU first drains the phase-0 jobs (formation of the first
// parent node: nothing can start before it); the TMA thread waits for ready[parent] before the
// first load of a tile; GEMM consumers count each stored tile into tiles_done[parent] and, when
// out of tiles, join the phase-1 queue.  All CTAs must be co-resident (cooperative launch,
// grid = #SMs), since jobs wait on tiles and tiles on jobs.
template <int BN, int WGM, int WGN, int STAGES, bool FUSED>
__global__ void __launch_bounds__(THREADS, 1)
    grouped_dgemm_tma(const GemmTask* __restrict__ tasks, const CUtensorMap* __restrict__ maps, int ntasks,
                      int total_tiles, Uniform uni, FusedArgs fa) {
  static_assert(WGM * WGN == CONSUMERS, "8 consumer warps");
  constexpr int WTM = BM / WGM, WTN = BN / WGN;
  static_assert(WTM % 16 == 0 && WTN % 16 == 0, "warp tile must be a multiple of 16");
  constexpr int MI = WTM / 8, NI = WTN / 8;
  constexpr int B_BYTES_T = BK * BN * 8;  // BN/16 boxes of 16 x 16
  constexpr int STAGE_T = A_BYTES + B_BYTES_T;
  extern __shared__ unsigned char smem_raw[];
  const unsigned raw = smem_u32(smem_raw);
  const unsigned al = (raw + 1023u) & ~1023u;  // 1024-byte alignment for the 128B swizzle
  // fused layout: [program area][barriers][pad to 1 KB][GEMM stages | worker staging]
  const unsigned sprog_u = al;
  const unsigned bars = FUSED ? al + FUSED_PROG_BYTES : al + STAGES * STAGE_T;
  const unsigned base = FUSED ? al + FUSED_HDR_BYTES : al;
  const char* sprog = reinterpret_cast<const char*>(smem_raw) + (sprog_u - raw);
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool adder = FUSED && (int)blockIdx.x >= fa.gemm_ctas;
  const int gemm_ctas = FUSED ? fa.gemm_ctas : (int)gridDim.x;

  if (threadIdx.x == 0) {
    if (!adder) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(full_bar(s), 1);
        mbar_init(empty_bar(s), CONSUMERS);
      }
    } else {
      for (int b = 0; b < 2 * ADD_WARPS; ++b) mbar_init(bars + 8u * b, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (FUSED) {  // the addition programs -> shared memory
    const int4* src = reinterpret_cast<const int4*>(fa.blob);
    int4* dst = reinterpret_cast<int4*>(smem_raw + (sprog_u - raw));
    for (int i = threadIdx.x; i < fa.blob_bytes / 16; i += THREADS) dst[i] = __ldg(src + i);
  }
  __syncthreads();

  if (FUSED && adder) {
    // ------------------------------ addition CTA ------------------------------
    Staging st;
    st.buf0 = base + (unsigned)(2 * warp) * FUSED_ADD_SEG_BYTES;
    st.bar0 = bars + 16u * warp;
    st.phase = 0;
    for (;;) {
      const int idx = claim(&fa.ctr[0], lane);
      if (idx >= fa.njobs0) break;
      run_job<4>(fa, sprog, idx, lane, &st);
    }
    for (;;) {
      const int idx = claim(&fa.ctr[1], lane);
      if (fa.njobs0 + idx >= fa.njobs) break;
      run_job<4>(fa, sprog, fa.njobs0 + idx, lane, &st);
    }
    return;
  }

  if (warp < 4) {
    // ------------------------------ producer warpgroup ------------------------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == 0 && lane == 0) {
      int stage = 0;
      unsigned phase = 0;
      int ready_node = -1;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gemm_ctas) {
        const TileCoord tc = locate<BN>(tasks, ntasks, tile, uni);
        if (FUSED) {
          const int node = __ldg(&tasks[tc.task].node);
          if (node != ready_node) {
            const unsigned long long target = (unsigned long long)__ldg(&fa.ready_target[node]);
            while (ld_acquire(&fa.ctr[2 + node]) < target) __nanosleep(128);
            fence_proxy_async_global();
            ready_node = node;
          }
        }
        const CUtensorMap* ma = maps + 2 * tc.task;
        const CUtensorMap* mb = ma + 1;
        const int KT = (__ldg(&tasks[tc.task].k) + BK - 1) / BK;
        for (int kt = 0; kt < KT; ++kt) {
          mbar_wait(empty_bar(stage), phase ^ 1u);
          const unsigned sa = base + stage * STAGE_T, sb = sa + A_BYTES;
          mbar_expect_tx(full_bar(stage), STAGE_T);
          tma_load_2d(sa, ma, kt * BK, tc.m0, full_bar(stage));
#pragma unroll
          for (int b = 0; b < BN / 16; ++b) tma_load_2d(sb + b * 2048, mb, tc.n0 + 16 * b, kt * BK, full_bar(stage));
          if (++stage == STAGES) stage = 0, phase ^= 1u;
        }
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");

  // ------------------------------ consumers ------------------------------
  if (FUSED) {
    for (;;) {
      const int idx = claim(&fa.ctr[0], lane);
      if (idx >= fa.njobs0) break;
      run_job<4>(fa, sprog, idx, lane, nullptr);
    }
  }
  const int cw = warp - 4;  // consumer warp 0..7
  const int r = lane >> 2, c = lane & 3;
  const int wm = (cw / WGN) * WTM, wn = (cw % WGN) * WTN;
  // A fragment: subtile i, fragment row r -> tile row R = wm + 16*(i/2) + 2r + (i%2);
  //   16-byte chunk = (2s + (c>>1)) ^ (R & 7); 8-byte half = c & 1
  const unsigned a_row0 = (unsigned)(wm + 2 * r) * 128u;
  const unsigned xa0 = (unsigned)((2 * r) & 7), xa1 = (unsigned)((2 * r + 1) & 7);
  const unsigned ha = (unsigned)(c & 1) * 8u, ca = (unsigned)(c >> 1);
  // B fragment: subtile jj, fragment col r -> box wn/16 + jj/2, box col 4*(jj%2) + map0[r];
  //   k row = 4s + c; chunk = (box col >> 1) ^ (k row & 7)
  const unsigned map0 = (r == 0) ? 0u : (r == 1) ? 1u : (r == 2) ? 8u : (r == 3) ? 9u : (r == 4) ? 2u : (r == 5) ? 3u : (r == 6) ? 10u : 11u;
  const unsigned hb = map0 & 1u, cb0 = map0 >> 1;
  const unsigned b_box0 = (unsigned)(wn / 16) * 2048u;

  int stage = 0;
  unsigned phase = 0;
  for (int tile = blockIdx.x; tile < total_tiles; tile += gemm_ctas) {
    const TileCoord tc = locate<BN>(tasks, ntasks, tile, uni);
    const GemmTask& t = tasks[tc.task];
    const int KT = (__ldg(&t.k) + BK - 1) / BK;
    // epilogue parameters, fetched now so their latency hides behind the main loop
    const double alpha = __ldg(&t.alpha), beta = __ldg(&t.beta);
    const int m = __ldg(&t.m), n = __ldg(&t.n);
    const long long ldc = __ldg(&t.ldc);
    double* C = t.C;
    double acc[MI][NI][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < KT; ++kt) {
      mbar_wait(full_bar(stage), phase);
      const unsigned sa = base + stage * STAGE_T, sb = sa + A_BYTES;
#pragma unroll
      for (int s = 0; s < BK / 4; ++s) {
        double a[MI], b[NI];
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const unsigned x = (i & 1) ? xa1 : xa0;
          const unsigned chunk = ((unsigned)(2 * s) + ca) ^ x;
          a[i] = lds64(sa + a_row0 + (unsigned)(16 * (i >> 1) + (i & 1)) * 128u + chunk * 16u + ha);
        }
        const unsigned krow = (unsigned)(4 * s + c);
#pragma unroll
        for (int jj = 0; jj < NI; ++jj) {
          const unsigned chunk = (cb0 + 2u * (jj & 1)) ^ (krow & 7u);
          b[jj] = lds64(sb + b_box0 + (unsigned)(jj >> 1) * 2048u + krow * 128u + chunk * 16u + hb * 8u);
        }
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int jj = 0; jj < NI; ++jj) dmma(acc[i][jj], a[i], b[jj]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_bar(stage));
      if (++stage == STAGES) stage = 0, phase ^= 1u;
    }

    // ---- epilogue: C = alpha * acc (+ beta * C), from registers ----
    const int cofs = (c == 0) ? 0 : (c == 1) ? 8 : (c == 2) ? 2 : 10;  // map0[2c]
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int row = tc.m0 + wm + 16 * (i >> 1) + 2 * r + (i & 1);
      if (row >= m) continue;
      double* crow = C + (long long)row * ldc;
#pragma unroll
      for (int jj = 0; jj < NI; ++jj) {
        const int col = tc.n0 + wn + 16 * (jj >> 1) + 4 * (jj & 1) + cofs;
        double v0 = alpha * acc[i][jj][0], v1 = alpha * acc[i][jj][1];
        if (col + 1 < n) {
          double2* p = reinterpret_cast<double2*>(crow + col);
          if (beta != 0.0) {
            const double2 o = *p;
            v0 = fma(beta, o.x, v0);
            v1 = fma(beta, o.y, v1);
          }
          *p = make_double2(v0, v1);
        } else if (col < n) {
          crow[col] = beta != 0.0 ? fma(beta, crow[col], v0) : v0;
        }
      }
    }
    if (FUSED) {  // publish the stored tile (release) to the assembly jobs of its parent
      __threadfence();
      named_bar_sync(1, CONSUMERS * 32);
      if (cw == 0 && lane == 0) atomicAdd(&fa.ctr[2 + fa.np + __ldg(&t.node)], 1ull);
    }
  }
  if (FUSED) {
    for (;;) {
      const int idx = claim(&fa.ctr[1], lane);
      if (fa.njobs0 + idx >= fa.njobs) break;
      run_job<4>(fa, sprog, fa.njobs0 + idx, lane, nullptr);
    }
  }
}

// ---- host side: tensor maps ----
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
    cudaGetLastError();
  });
  return fn;
}

void make_map(CUtensorMap* m, const double* ptr, long long rows, long long cols, long long ld, int box_cols, int box_rows) {
  EncodeFn fn = encode_fn();
  if (!fn) throw Error(FMM_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)std::max<long long>(cols, 1), (cuuint64_t)std::max<long long>(rows, 1)};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(FMM_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}
}  // namespace

size_t gemm_tma_map_bytes() { return sizeof(CUtensorMap); }

bool gemm_tma_eligible(const std::vector<GemmTask>& tasks) {
  if (!encode_fn()) return false;
  for (const auto& t : tasks) {
    if ((reinterpret_cast<uintptr_t>(t.A) & 15) || (reinterpret_cast<uintptr_t>(t.B) & 15)) return false;
    if ((t.lda & 1) || (t.ldb & 1) || (t.ldc & 1) || (reinterpret_cast<uintptr_t>(t.C) & 15)) return false;
  }
  return true;
}

void gemm_tma_maps(const std::vector<GemmTask>& tasks, void* out) {
  auto* maps = reinterpret_cast<CUtensorMap*>(out);
  for (size_t i = 0; i < tasks.size(); ++i) {
    const GemmTask& t = tasks[i];
    make_map(&maps[2 * i], t.A, t.m, t.k, t.lda, BK, BM);      // A view: m rows x k cols, box 128 x 16
    make_map(&maps[2 * i + 1], t.B, t.k, t.n, t.ldb, 16, BK);  // B view: k rows x n cols, box 16 x 16
  }
}

template <int BN, int WGM, int WGN, bool FUSED>
static void launch_cfg(const GemmTask* d_tasks, const void* d_maps, int ntasks, long long total_tiles, int sms,
                       Uniform uni, const FusedArgs& fa, cudaStream_t stream) {
  constexpr int ST = FUSED ? STAGES_FUSED : STAGES_PLAIN;
  static bool configured = false;  // per process; one device per process (torchrun)
  auto kern = grouped_dgemm_tma<BN, WGM, WGN, ST, FUSED>;
  const size_t smem = smem_bytes(BN, ST, FUSED);
  if (!configured) {
    FMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  const CUtensorMap* maps = reinterpret_cast<const CUtensorMap*>(d_maps);
  const int ntiles = (int)total_tiles;
  if (!FUSED) {
    const int grid = (int)std::min<long long>(total_tiles, sms);
    kern<<<grid, THREADS, smem, stream>>>(d_tasks, maps, ntasks, ntiles, uni, fa);
    FMM_CUDA(cudaGetLastError());
    return;
  }
  // fused: every SM hosts addition workers, and assembly jobs wait on tiles of other CTAs, so all
  // CTAs must be co-resident: cooperative launch, one CTA per SM
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)sms);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  FMM_CUDA(cudaLaunchKernelEx(&cfg, kern, d_tasks, maps, ntasks, ntiles, uni, fa));
}

int gemm_choose_bn(const std::vector<GemmTask>& tasks) {
  if (const char* e = getenv("FMM_GEMM_BN")) return atoi(e);
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
    cudaGetLastError();
  }
  // relative DMMA efficiency of each tile width (narrow tiles read more operand bytes per flop)
  static const int menu[] = {128, 112, 96, 80, 64};
  static const double eff[] = {1.00, 0.985, 0.975, 0.965, 0.94};
  int best = 128;
  double best_t = 1e300;
  for (int q = 0; q < 5; ++q) {
    const int bn = menu[q];
    double work = 0, tiles = 0;
    for (const auto& t : tasks) {
      const double tl = (double)((t.m + BM - 1) / BM) * ((t.n + bn - 1) / bn);
      tiles += tl;
      work += tl * BM * bn * (double)(((t.k + BK - 1) / BK) * BK + 32 /* epilogue, prologue */);
    }
    if (tiles <= 0) continue;
    const double waves = std::ceil(tiles / sms);
    const double tmax = std::max(work / tiles * waves, work / sms);  // per-SM time, unit work
    const double t_est = tmax / eff[q];
    if (t_est < best_t * 0.999) best_t = t_est, best = bn;
  }
  return best;
}

static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    FMM_CUDA(cudaGetDevice(&dev));
    FMM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return sms;
}

template <bool FUSED>
static void launch_bn(const GemmTask* d_tasks, const void* d_maps, int ntasks, long long total_tiles, int bn, Uniform uni,
                      const FusedArgs& fa, cudaStream_t stream) {
  const int sms = sm_count();
  switch (bn) {
    case 128: launch_cfg<128, 2, 4, FUSED>(d_tasks, d_maps, ntasks, total_tiles, sms, uni, fa, stream); break;
    case 112: launch_cfg<112, 8, 1, FUSED>(d_tasks, d_maps, ntasks, total_tiles, sms, uni, fa, stream); break;
    case 96: launch_cfg<96, 4, 2, FUSED>(d_tasks, d_maps, ntasks, total_tiles, sms, uni, fa, stream); break;
    case 80: launch_cfg<80, 8, 1, FUSED>(d_tasks, d_maps, ntasks, total_tiles, sms, uni, fa, stream); break;
    case 64: launch_cfg<64, 4, 2, FUSED>(d_tasks, d_maps, ntasks, total_tiles, sms, uni, fa, stream); break;
    default: throw Error(FMM_E_INVALID_ARG, "unsupported GEMM tile width " + std::to_string(bn));
  }
}

void gemm_tma_launch(const GemmTask* d_tasks, const void* d_maps, int ntasks, long long total_tiles, int bn,
                     int uniform_tm, int uniform_tn, cudaStream_t stream) {
  const Uniform uni{uniform_tm * uniform_tn, uniform_tm, uniform_tn};
  if (total_tiles <= 0 || ntasks <= 0) return;
  launch_bn<false>(d_tasks, d_maps, ntasks, total_tiles, bn, uni, FusedArgs{}, stream);
}

void gemm_fused_launch(const GemmTask* d_tasks, const void* d_maps, int ntasks, long long total_tiles, int bn,
                       int uniform_tm, int uniform_tn, const FusedArgs& fa, cudaStream_t stream) {
  const Uniform uni{uniform_tm * uniform_tn, uniform_tm, uniform_tn};
  if (ntasks <= 0 && fa.njobs <= 0) return;
  launch_bn<true>(d_tasks, d_maps, ntasks, total_tiles, bn, uni, fa, stream);
}

}  // namespace fmm
