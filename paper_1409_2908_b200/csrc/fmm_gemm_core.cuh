// GEMM core of K2 (and of the fused leaf level): persistent, warp-specialised grouped FP64 GEMM
// fed by TMA.  Included by fmm_gemm_tma.cu (nvcc, the plain kernels) and embedded verbatim into
// the NVRTC source of the fused leaf-level kernel (fmm_codegen.cpp), so it has no includes.
//
// Per CTA (one per SM, looping over tiles):
//   warpgroup 0 (producer): one thread issues cp.async.bulk.tensor (TMA) loads of the A tile
//       (one 128x16 box) and the B tile (BN/16 boxes of 16x16) per k-step into a 6-stage ring of
//       shared-memory buffers as soon as a stage is released, signalling a "full" mbarrier with
//       complete_tx; it runs over the CTA's whole (tile, k-step) sequence, so the next tile's
//       loads are in flight while the current tile's epilogue runs.  It gives its registers
//       away with setmaxnreg.dec (40), so the consumers can grow to 232 (setmaxnreg.inc) --
//       the 64x32 warp tile needs ~210, above the 168 a flat 384-thread launch would allow.
//   warpgroups 1-2 (consumers): 8 warps of (128/WGM) x (BN/WGN) outputs; wait "full", read
//       register fragments, issue mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), arrive "empty";
//       epilogue straight from registers with 16-byte stores.  No CTA-wide barrier in the loop.
// TMA writes the tiles with the 128-byte swizzle (16-byte chunk index XOR row mod 8).  The DMMA
// fragment pattern (lane -> row lane/4, col lane%4 for A; row lane%4, col lane/4 for B) would hit
// 2- or 4-way bank conflicts on that layout, so fragment rows and columns are mapped to tile rows
// and columns by fixed permutations chosen to make every 8-byte fragment load conflict-free:
//   A: fragment row r of m-subtile i  -> tile row 16*(i/2) + 2r + (i%2)
//   B: fragment col j of n-subtile jj -> tile col 16*(jj/2) + 4*(jj%2) + {0,1,8,9,2,3,10,11}[j]
// The epilogue writes each accumulator to the tile position its operands came from.
//
// FUSED (NVRTC only): the level-L formation (F) and assembly (A) jobs of a plan run in the same
// launch, spatially partitioned: CTAs [0, gemm_ctas) run leaf tiles exactly as above, CTAs
// [gemm_ctas, gridDim.x) are addition CTAs whose 12 warps run the plan's generated addition
// chains (fmm_add_job, straight-line code from fmm_codegen.cpp).  They must not share an SM: the
// FP64 ALU (DADD) and the DMMA path are one pipe on B200, and a DADD warp beside eight DMMA warps
// was measured to crawl.  Every warp of the GPU first drains the phase-0 jobs (formation of the
// first parent: nothing can start before it); the TMA thread waits for ready[parent] before the
// first load of a tile; consumers count each stored tile into tiles_done[parent] and, out of
// tiles, join the phase-1 queue.  All CTAs must be co-resident (cooperative launch, grid = #SMs):
// jobs wait on tiles and tiles on jobs.  FMM_FUSED_BG (background mode): no addition CTAs; warps
// 1-3 of every CTA's producer warpgroup run the jobs (staged through shared memory, 56 registers)
// beside the CTA's own leaf tiles -- correct, but the DADDs starve beside DMMA.
#pragma once

namespace fmm {

#ifdef FMM_NVRTC
struct alignas(64) CUtensorMap_opaque {
  unsigned long long opaque[16];
};
typedef CUtensorMap_opaque CUtensorMap;
#endif

// BK: k-depth of a ring stage of the fused leaf level and K3f; the plain kernel is instantiated for
// k-steps KS = 16, 32 and 48 (KS/4 4-deep slices per stage: A as KS/16 boxes of 128 x 16, B as
// boxes of KS x 16): fewer stage hand-overs per flop with about the same bytes in flight
#ifndef FMM_GEMM_BK
#define FMM_GEMM_BK 16
#endif
constexpr int BM = 128, BK = FMM_GEMM_BK;
static_assert(BK == 16 || BK == 32, "a stage holds one or two 16-column A boxes");
#ifndef FMM_F1_EMUL_U
#define FMM_F1_EMUL_U 1
#endif
#ifndef FMM_F1_EMUL_V
#define FMM_F1_EMUL_V 1
#endif
#ifndef FMM_GEMM_STAGES
#define FMM_GEMM_STAGES 6  // of 16-deep stages; 32-deep rings have half as many
#endif
// 16-deep: FMM_GEMM_STAGES stages; 32-deep: half as many; 48-deep: two (96 KB of k in flight)
__host__ __device__ constexpr int ring_stages(int ks) { return ks >= 48 ? 2 : FMM_GEMM_STAGES * 16 / ks; }
constexpr int GEMM_STAGES = ring_stages(BK);
constexpr int CONSUMERS = 8, THREADS = 128 + CONSUMERS * 32;  // warpgroup 0 = producer, 1-2 = consumers
static_assert(THREADS == GEMM_THREADS, "host and device agree on the block size");
constexpr int A_BYTES = BM * BK * 8;                           // 16 KB per 16 columns of k
__host__ __device__ constexpr int gemm_smem_bytes(int bn, int ks = BK) {
  return ring_stages(ks) * (BM * ks * 8 + ks * bn * 8) + 1024 /*align*/ + 256 /*barriers*/;
}
// Staged epilogue (EPI = 1): four staging slots, one per SM sub-partition, each shared by the two
// consumer warps of that sub-partition in turn; a slot holds one warp tile (row stride padded by
// 16 bytes: conflict-free 16-byte fragment stores).  The ring keeps as many stages as fit beside it.
constexpr int SMEM_OPTIN = 232448;
__host__ __device__ constexpr int epi_stride(int bn, int wgn) { return (bn / wgn) * 8 + 16; }
__host__ __device__ constexpr int epi_slot_bytes(int bn, int wgm, int wgn) { return (BM / wgm) * epi_stride(bn, wgn); }
__host__ __device__ constexpr int epi_ring_stages(int ks, int bn, int wgm, int wgn, int slots = 4) {
  return (SMEM_OPTIN - 1024 - 256 - slots * epi_slot_bytes(bn, wgm, wgn)) / (BM * ks * 8 + ks * bn * 8) < ring_stages(ks)
             ? (SMEM_OPTIN - 1024 - 256 - slots * epi_slot_bytes(bn, wgm, wgn)) / (BM * ks * 8 + ks * bn * 8)
             : ring_stages(ks);
}
__host__ __device__ constexpr int gemm_epi_smem_bytes(int bn, int ks, int wgm, int wgn, int slots = 4) {
  return epi_ring_stages(ks, bn, wgm, wgn, slots) * (BM * ks * 8 + ks * bn * 8) + 1024 + 256 +
         slots * epi_slot_bytes(bn, wgm, wgn);
}
// bg_stage: per producer warp, the background jobs' input staging (3 warps)
__host__ __device__ constexpr int fused_smem_bytes(int bn, int ks = BK, int bg_stage = 0) {
  return gemm_smem_bytes(bn, ks) + FUSED_PTR_BYTES + 3 * bg_stage;
}
#ifndef FMM_BG_STAGE_W
#define FMM_BG_STAGE_W 0
#endif
// K3f: a 4-stage ring plus two staging tiles (+alpha acc and -alpha acc) of 128 x bn doubles
constexpr int K3F_STAGES = 64 / BK;
__host__ __device__ constexpr int k3f_smem_bytes(int bn) {
  return K3F_STAGES * (A_BYTES + BK * bn * 8) + 1024 /*align*/ + 1024 /*barriers, aligned*/ + 2 * BM * bn * 8;
}
#ifndef FMM_GROUP_M
#define FMM_GROUP_M 8  // row tiles per raster group (tiles of a group run column by column)
#endif
constexpr int GROUP_M = FMM_GROUP_M;
// FMM_FUSED_BG (fused kernel only): every CTA runs leaf tiles and the producer warpgroup's warps
// 1-3 run the addition jobs beside them (no addition CTAs)
#ifndef FMM_FUSED_BG
#define FMM_FUSED_BG 0
#endif
// register split of the warp-specialised CTA (setmaxnreg).  The CTA is launched with 168 registers
// per thread (__launch_bounds__(384, 1)); setmaxnreg.inc blocks until the producer's .dec has
// returned enough of them, so the split must fit what the CTA holds: 128 P + 256 C <= 384 x 168
#ifndef FMM_PRODUCER_REGS
#define FMM_PRODUCER_REGS 40
#endif
#ifndef FMM_CONSUMER_REGS
#define FMM_CONSUMER_REGS 232
#endif
static_assert(128 * FMM_PRODUCER_REGS + 256 * FMM_CONSUMER_REGS <= 384 * 168,
              "register split exceeds the CTA's allocation (setmaxnreg.inc would wait forever)");

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
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// Experiments (off by default): FMM_L2_HINT=1 loads the operand tiles with an L2
// evict_last policy, so the streaming output does not push operand panels that other SMs still read
// out of L2 (DRAM re-reads on c2 / c5); FMM_GEMM_STG=1 stores the epilogue through st.global
// (STG) instead of the generic ST the compiler emits for C, =2 through st.global.cs (evict-first)
#ifndef FMM_L2_HINT
#define FMM_L2_HINT 0
#endif
#ifndef FMM_GEMM_STG
#define FMM_GEMM_STG 0
#endif
__device__ __forceinline__ void st_global_v2(double2* p, double a, double b) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};\n" ::"l"(p), "d"(a), "d"(b) : "memory");
}
__device__ __forceinline__ void tma_load_2d_hint(unsigned dst, const CUtensorMap* map, int c0, int c1, unsigned bar,
                                                 unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;\n" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ unsigned long long l2_policy_evict_last() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_shared() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// K3f: shared-memory box (16 columns x 128 rows, 128B swizzle) reduce-added into a global tile
__device__ __forceinline__ void tma_reduce_add_2d(const void* map, int c0, int c1, unsigned src) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
          reinterpret_cast<unsigned long long>(map)),
      "r"(c0), "r"(c1), "r"(src)
      : "memory");
}
// staged epilogue: one row of a warp tile, shared memory -> global, by the bulk-copy engine
__device__ __forceinline__ void bulk_store(double* dst, unsigned src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void sts_f64x2(unsigned addr, double a, double b) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(addr), "d"(a), "d"(b) : "memory");
}
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
__device__ __forceinline__ unsigned long long lds_u64(unsigned addr) {
  unsigned long long v;
  asm volatile("ld.shared.u64 %0, [%1];\n" : "=l"(v) : "r"(addr));
  return v;
}
// background jobs: each lane stages its element's inputs in shared memory (no registers held while
// the copies are in flight), 8 bytes per lane per input
__device__ __forceinline__ void cp_async8(unsigned dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void sts_u64(unsigned addr, unsigned long long v) {
  asm volatile("st.shared.u64 [%0], %1;\n" ::"r"(addr), "l"(v) : "memory");
}
// Loads of the addition jobs.  Assembly inputs are written by other SMs during this kernel; the
// job's lane 0 acquires the tile counter first (ld.acquire.gpu, which invalidates this SM's L1)
// and the warp synchronises, so weak loads after it see the stored tiles.  FMM_LD_KIND selects the
// flavour: 0 = ld.global.cg (L2 only), 1 = ld.global (L1-allocating), 2 = ld.global.nc.
#ifndef FMM_LD_KIND
#define FMM_LD_KIND 0
#endif
__device__ __forceinline__ double2 ldcg2(const double* p) {
  double2 v;
#if FMM_LD_KIND == 0
  asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
#elif FMM_LD_KIND == 1
  v = *reinterpret_cast<const double2*>(p);
#else
  v = __ldg(reinterpret_cast<const double2*>(p));
#endif
  return v;
}
__device__ __forceinline__ double ldcg1(const double* p) {
  double v;
#if FMM_LD_KIND == 0
  asm volatile("ld.global.cg.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
#elif FMM_LD_KIND == 1
  v = *p;
#else
  v = __ldg(p);
#endif
  return v;
}

struct TileCoord {
  int task, m0, n0;
};
// x / d for 0 <= x < 2^31 with magic = floor((2^32 - 1) / d): the multiply-high estimate is the
// quotient or one below it, so one correction makes it exact
__device__ __forceinline__ int magic_div(int x, int d, unsigned magic, int& rem) {
  unsigned q = __umulhi((unsigned)x, magic);
  unsigned r = (unsigned)x - q * (unsigned)d;
  if (r >= (unsigned)d) ++q, r -= (unsigned)d;
  rem = (int)r;
  return (int)q;
}

template <int BN>
__device__ __forceinline__ TileCoord locate(const GemmTask* __restrict__ tasks, int ntasks, int tile, Uniform u) {
  int lo, tiles_m, tiles_n, local;
  if (u.tiles) {
    if (u.magic_tiles) {
      lo = magic_div(tile, u.tiles, u.magic_tiles, local);
    } else {
      lo = tile / u.tiles;
      local = tile - lo * u.tiles;
    }
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
  int group, in_span;
  if (u.tiles && u.magic_span) {
    group = magic_div(local, span, u.magic_span, in_span);
  } else {
    group = local / span;
    in_span = local - group * span;
  }
  const int first_m = group * GROUP_M;
  const int gsize = min(tiles_m - first_m, GROUP_M);
  int tn, tm_in;
  if (gsize == GROUP_M) {  // every group but a ragged last one: a compile-time divisor
    tn = in_span / GROUP_M;
    tm_in = in_span % GROUP_M;
  } else {
    tn = in_span / gsize;
    tm_in = in_span - tn * gsize;
  }
  return {lo, (first_m + tm_in) * BM, tn * BN};
}


__device__ __forceinline__ int claim(unsigned long long* ctr, int lane) {
  int idx = 0;
  if (lane == 0) idx = (int)atomicAdd(ctr, 1ull);
  return __shfl_sync(0xffffffffu, idx, 0);
}

// Generated per algorithm (fmm_codegen.cpp) in the NVRTC source of the fused kernel.
// sp: shared address of the warp's FUSED_PTR_SLOT.
__device__ void fmm_add_job(const FusedArgs& fa, const FusedJob& j, int lane, unsigned sp);
// background mode: the same chains with the inputs staged at st (FMM_BG_STAGE_W bytes of shared memory)
__device__ void fmm_add_job_bg(const FusedArgs& fa, const FusedJob& j, int lane, unsigned sp, unsigned st);

// One job with a whole warp: assembly jobs first wait until every leaf tile of their parent is
// stored; formation jobs publish (release) to the TMA readers of the leaf products.
// FMM_FUSED_STATS (diagnostics): clock64 totals in ctr[2 + 2 np + i]: 0 the TMA threads' waits for
// formation, 1 the assembly jobs' waits for tiles, 2 / 3 job time in producer / consumer warps
#ifndef FMM_FUSED_STATS
#define FMM_FUSED_STATS 0
#endif
template <bool STAGED = false>
__device__ __forceinline__ void run_job(const FusedArgs& fa, int jidx, int lane, unsigned sp, unsigned st = 0) {
  const FusedJob j = fa.jobs[jidx];
#if FMM_FUSED_STATS
  const long long t0 = clock64();
#endif
  if (j.kind == 1) {
    if (lane == 0) {
      const unsigned long long target = (unsigned long long)__ldg(&fa.tiles_target[j.dep]);
      while (ld_acquire(&fa.ctr[2 + fa.np + j.dep]) < target) __nanosleep(256);
      fence_proxy_async_global();  // the tiles were stored by generic proxies; TMA reads them
#if FMM_FUSED_STATS
      atomicAdd(&fa.ctr[2 + 2 * fa.np + 1], (unsigned long long)(clock64() - t0));
#endif
    }
    __syncwarp();
  }
  if constexpr (STAGED) fmm_add_job_bg(fa, j, lane, sp, st);
  else fmm_add_job(fa, j, lane, sp);
  if (j.kind == 0) {
    fence_proxy_async_global();
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicAdd(&fa.ctr[2 + j.dep], 1ull);
  }
#if FMM_FUSED_STATS
  if (lane == 0) atomicAdd(&fa.ctr[2 + 2 * fa.np + (STAGED ? 2 : 3)], (unsigned long long)(clock64() - t0));
#endif
}

#ifdef FMM_BG_PROBE
__device__ const double* fmm_bg_src;
__device__ double* fmm_bg_dst;
__device__ long long fmm_bg_n;
#endif
template <int BN, int WGM, int WGN, bool FUSED, bool K3F = false, int KS = BK, int EPI = 0>
__device__ __forceinline__ void gemm_body(const GemmTask* __restrict__ tasks, const CUtensorMap* __restrict__ maps,
                                          int ntasks, int total_tiles, Uniform uni, const FusedArgs& fa,
                                          const K3fArgs* ka = nullptr) {
  static_assert(!(FUSED && K3F), "one epilogue mode");
  static_assert(KS == 16 || KS == 32 || KS == 48, "16-, 32- or 48-deep stages (whole 16-column A boxes)");
  static_assert(KS == BK || !K3F, "the K3f kernel uses BK-deep stages");
  static_assert(!EPI || (!FUSED && !K3F), "the staged epilogue is the plain kernel's");
  constexpr int STAGES = K3F ? K3F_STAGES : EPI ? epi_ring_stages(KS, BN, WGM, WGN, EPI == 2 ? 8 : 4) : ring_stages(KS);
  static_assert(STAGES >= 2, "at least two ring stages");
  constexpr int A_BYTES = BM * KS * 8;
  static_assert(WGM * WGN == CONSUMERS, "8 consumer warps");
  constexpr int WTM = BM / WGM, WTN = BN / WGN;
  static_assert(WTM % 16 == 0 && WTN % 16 == 0, "warp tile must be a multiple of 16");
  constexpr int MI = WTM / 8, NI = WTN / 8;
  constexpr int B_BYTES_T = KS * BN * 8;  // BN/16 boxes of KS x 16
  constexpr int B_BOX = KS * 128;          // bytes of one B box (KS rows of 16 doubles)
  constexpr int SL = KS / 4;               // 4-deep slices per stage
  constexpr int STAGE_T = A_BYTES + B_BYTES_T;
  extern __shared__ unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned raw = smem_u32(smem_raw);
  const unsigned base = (raw + 1023u) & ~1023u;  // 1024-byte alignment for the 128B swizzle
  const unsigned bars = base + STAGES * STAGE_T;
  const unsigned sp = bars + 256u + (unsigned)warp * FUSED_PTR_SLOT;  // fused: this warp's pointer slot
  int gemm_ctas = (int)gridDim.x;
#if !FMM_FUSED_BG
  if constexpr (FUSED) {
    gemm_ctas = fa.gemm_ctas;
    if ((int)blockIdx.x >= gemm_ctas) {
      // ------------------------------ addition CTA ------------------------------
      for (;;) {
        const int idx = claim(&fa.ctr[0], lane);
        if (idx >= fa.njobs0) break;
        run_job(fa, idx, lane, sp);
      }
      for (;;) {
        const int idx = claim(&fa.ctr[1], lane);
        if (fa.njobs0 + idx >= fa.njobs) break;
        run_job(fa, fa.njobs0 + idx, lane, sp);
      }
      return;
    }
  }
#endif
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp < 4) {
    // ------------------------------ producer warpgroup ------------------------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(FMM_PRODUCER_REGS) : "memory");
    if (warp == 0 && lane == 0) {
      int stage = 0;
      unsigned phase = 0;
      int ready_node = -1;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gemm_ctas) {
        const TileCoord tc = locate<BN>(tasks, ntasks, tile, uni);
        if constexpr (FUSED) {
          const int node = __ldg(&tasks[tc.task].node);
          if (node != ready_node) {
            // (a watchdog __trap() in these waits was measured to slow the whole launch by ~13 %)
            const unsigned long long target = (unsigned long long)__ldg(&fa.ready_target[node]);
#if FMM_FUSED_STATS
            const long long t0 = clock64();
#endif
            while (ld_acquire(&fa.ctr[2 + node]) < target) __nanosleep(128);
#if FMM_FUSED_STATS
            atomicAdd(&fa.ctr[2 + 2 * fa.np], (unsigned long long)(clock64() - t0));
#endif
            fence_proxy_async_global();
            ready_node = node;
          }
        }
        const CUtensorMap* ma = maps + 2 * tc.task;
        const CUtensorMap* mb = ma + 1;
        const int KT = (__ldg(&tasks[tc.task].k) + KS - 1) / KS;
        for (int kt = 0; kt < KT; ++kt) {
          mbar_wait(empty_bar(stage), phase ^ 1u);
          const unsigned sa = base + stage * STAGE_T, sb = sa + A_BYTES;
          mbar_expect_tx(full_bar(stage), STAGE_T);
#if FMM_L2_HINT
          const unsigned long long pol = l2_policy_evict_last();
#pragma unroll
          for (int h = 0; h < KS / 16; ++h)
            tma_load_2d_hint(sa + h * 16384, ma, kt * KS + 16 * h, tc.m0, full_bar(stage), pol);
#pragma unroll
          for (int b = 0; b < BN / 16; ++b)
            tma_load_2d_hint(sb + b * B_BOX, mb, tc.n0 + 16 * b, kt * KS, full_bar(stage), pol);
#else
#pragma unroll
          for (int h = 0; h < KS / 16; ++h) tma_load_2d(sa + h * 16384, ma, kt * KS + 16 * h, tc.m0, full_bar(stage));
#pragma unroll
          for (int b = 0; b < BN / 16; ++b) tma_load_2d(sb + b * B_BOX, mb, tc.n0 + 16 * b, kt * KS, full_bar(stage));
#endif
          if (++stage == STAGES) stage = 0, phase ^= 1u;
        }
      }
    }
#if FMM_FUSED_BG
    // background mode: the producer warpgroup's idle warps 1-3 run the addition jobs while the
    // consumers run the leaf tiles of the same SM (the first parent's formation with every warp)
    if constexpr (FUSED) {
      if (warp >= 1) {
        const unsigned st = bars + 256u + FUSED_PTR_BYTES + (unsigned)(warp - 1) * FMM_BG_STAGE_W;
        for (;;) {
          const int idx = claim(&fa.ctr[0], lane);
          if (idx >= fa.njobs0) break;
          run_job<true>(fa, idx, lane, sp, st);
        }
        for (;;) {
          const int idx = claim(&fa.ctr[1], lane);
          if (fa.njobs0 + idx >= fa.njobs) break;
          run_job<true>(fa, fa.njobs0 + idx, lane, sp, st);
        }
      }
    }
#endif
#ifdef FMM_BG_PROBE  // timing experiment: the producer warpgroup's idle warps 1-3 stream-copy a buffer
    // (read + write, 16-byte accesses, 4 in flight per lane) while the consumers run the GEMM: the
    // cost of background bandwidth work inside GEMM CTAs (results of the copy are not used)
    if constexpr (!FUSED && !K3F) {
      if (warp >= 1 && fmm_bg_n > 0) {
        const long long n2 = fmm_bg_n / 2;
        const long long tid = (long long)blockIdx.x * 96 + (warp - 1) * 32 + lane, nth = (long long)gridDim.x * 96;
        const double2* src = reinterpret_cast<const double2*>(fmm_bg_src);
        double2* dst = reinterpret_cast<double2*>(fmm_bg_dst);
        long long e = tid;
        for (; e + 3 * nth < n2; e += 4 * nth) {
          double2 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = __ldcs(src + e + u * nth);
#pragma unroll
          for (int u = 0; u < 4; ++u) __stcs(dst + e + u * nth, v[u]);
        }
        for (; e < n2; e += nth) __stcs(dst + e, __ldcs(src + e));
      }
    }
#endif
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(FMM_CONSUMER_REGS) : "memory");

  // ------------------------------ consumers ------------------------------
  if constexpr (FUSED) {
    for (;;) {
      const int idx = claim(&fa.ctr[0], lane);
      if (idx >= fa.njobs0) break;
      run_job(fa, idx, lane, sp);
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
  const unsigned b_box0 = (unsigned)(wn / 16) * (unsigned)B_BOX;

  int stage = 0;
  unsigned phase = 0;
  // The tile -> (task, m0, n0) map (three integer divisions, or a binary search) of the NEXT tile
  // is computed inside the current tile's main loop, where issue slots are idle behind the DMMAs;
  // the two warps of a sub-partition do it in different k-steps so one of them keeps the pipe fed.
  // Measured (profiles/r2_fast_epilogue_study.jsonl): 112-wide tiles gain (c3 0.930 -> 0.933, c4 0.937 ->
  // 0.945 of the DMMA peak); 80-wide tiles lose (ptxas spills two registers into the main loop: c5t
  // 0.935 -> 0.924, c5 0.966 -> 0.958) and 128-wide tiles are unchanged, so only BN = 112 does it.
  constexpr bool NEXT_IN_LOOP = BN == 112;
  TileCoord tc_next = locate<BN>(tasks, ntasks, (int)blockIdx.x < total_tiles ? (int)blockIdx.x : 0, uni);
  for (int tile = blockIdx.x; tile < total_tiles; tile += gemm_ctas) {
    const TileCoord tc = tc_next;
    const int tile_next = tile + gemm_ctas;
    bool have_next = false;
    const GemmTask& t = tasks[tc.task];
    const int kdim = __ldg(&t.k);
    const int KT = (kdim + KS - 1) / KS;
    // epilogue parameters, fetched now so their latency hides behind the main loop
    const double alpha = __ldg(&t.alpha), beta = __ldg(&t.beta);
    const int m = __ldg(&t.m), n = __ldg(&t.n);
    // ragged edge tiles: a warp whose sub-tile lies beyond m or n may skip its DMMAs.  That only
    // shortens the tile when every SM sub-partition loses work (consumer warps cw and cw + 4 share
    // one), so warps skip only when no sub-partition keeps both of its warps busy; otherwise all run
    // (zero fill costs nothing extra there, and a lone early warp was measured to cost ~1 %).
    auto in_range = [&](int w) { return (tc.m0 + (w / WGN) * WTM < m) && (tc.n0 + (w % WGN) * WTN < n); };
    bool full_pair = false;
#pragma unroll
    for (int q = 0; q < CONSUMERS / 2; ++q) full_pair |= in_range(q) && in_range(q + CONSUMERS / 2);
    const bool active = full_pair || in_range(cw);
    const long long ldc = __ldg(&t.ldc);
    double* C = t.C;
    double acc[MI][NI][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // fragments of one 4-deep k-slice from shared memory, and its MI x NI DMMAs
    auto load = [&](double (&a)[MI], double (&b)[NI], unsigned sa, unsigned sb, int s) {
      const unsigned sa_h = sa + (unsigned)(s >> 2) * 16384u;  // the A box of this slice's 16 columns
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const unsigned x = (i & 1) ? xa1 : xa0;
        const unsigned chunk = ((unsigned)(2 * (s & 3)) + ca) ^ x;
        const unsigned off = a_row0 + (unsigned)(16 * (i >> 1) + (i & 1)) * 128u + chunk * 16u + ha + (sa_h - sa);
        a[i] = lds64(sa + off);
#if FMM_F1_EMUL_U > 1  // timing experiment: a leaf operand formed in registers from
        // FMM_F1_EMUL_U parent tiles -- extra fragment loads (other rows of the same stage, so the
        // bank pattern is unchanged) and DADDs on the FP64 pipe the DMMAs use; results are wrong
#pragma unroll
        for (int q = 1; q < FMM_F1_EMUL_U; ++q) a[i] = a[i] + lds64(sa + ((off + 2048u * q) & (unsigned)(A_BYTES - 1)));
#endif
      }
      const unsigned krow = (unsigned)(4 * s + c);
#pragma unroll
      for (int jj = 0; jj < NI; ++jj) {
        const unsigned chunk = (cb0 + 2u * (jj & 1)) ^ (krow & 7u);
        const unsigned off = b_box0 + (unsigned)(jj >> 1) * (unsigned)B_BOX + krow * 128u + chunk * 16u + hb * 8u;
        b[jj] = lds64(sb + off);
#if FMM_F1_EMUL_V > 1
#pragma unroll
        for (int q = 1; q < FMM_F1_EMUL_V; ++q) {
          unsigned o2 = off + 2048u * q;
          while (o2 >= (unsigned)B_BYTES_T) o2 -= (unsigned)B_BYTES_T;
          b[jj] = b[jj] + lds64(sb + o2);
        }
#endif
      }
    };
    auto mma = [&](const double (&a)[MI], const double (&b)[NI]) {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int jj = 0; jj < NI; ++jj) dmma(acc[i][jj], a[i], b[jj]);
    };
    auto release = [&]() {
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_bar(stage));
      if (++stage == STAGES) stage = 0, phase ^= 1u;
    };
    // Full stages: software-pipelined -- the fragments of slice s + 1 (for the last slice, slice 0
    // of the next stage, after its full barrier) are loaded before the DMMAs of slice s, so the
    // shared-memory latency hides behind the warp's own DMMAs, not only behind the other warp of
    // its sub-partition.  A stage is released after the DMMAs that consume its last fragments.
    // Then a ragged last k-step runs only the 4-deep slices that hold data (the rest is zero fill),
    // and a warp whose sub-tile lies beyond m or n (ragged edge tiles) issues no DMMA at all but
    // waits for and releases every stage with the others.
    const int KF = active ? kdim / KS : 0;
    if (KF > 0) {
      static_assert(SL % 2 == 0, "slices come in pairs");
      double a0[MI], b0[NI], a1[MI], b1[NI];
      mbar_wait(full_bar(stage), phase);
      unsigned sa = base + stage * STAGE_T, sb = sa + A_BYTES;
      load(a0, b0, sa, sb, 0);
      const int pfk = min(cw >= CONSUMERS / 2 ? 1 : 0, KF - 1);
      for (int kt = 0; kt < KF; ++kt) {
        if (NEXT_IN_LOOP && kt == pfk) {
          if (tile_next < total_tiles) tc_next = locate<BN>(tasks, ntasks, tile_next, uni);
          have_next = true;
        }
#pragma unroll
        for (int s = 0; s + 2 < SL; s += 2) {
          load(a1, b1, sa, sb, s + 1);
          mma(a0, b0);
          load(a0, b0, sa, sb, s + 2);
          mma(a1, b1);
        }
        load(a1, b1, sa, sb, SL - 1);
        mma(a0, b0);
        if (kt + 1 < KF) {
          const int nx = stage + 1 == STAGES ? 0 : stage + 1;
          mbar_wait(full_bar(nx), nx == 0 ? phase ^ 1u : phase);
          sa = base + nx * STAGE_T, sb = sa + A_BYTES;
          load(a0, b0, sa, sb, 0);
        }
        mma(a1, b1);
        release();
      }
    }
    for (int kt = KF; kt < KT; ++kt) {
      mbar_wait(full_bar(stage), phase);
      const unsigned sa = base + stage * STAGE_T, sb = sa + A_BYTES;
      const int ks = active ? (kdim - kt * KS + 3) / 4 : 0;
#pragma unroll 1
      for (int s = 0; s < ks; ++s) {
        double a[MI], b[NI];
        load(a, b, sa, sb, s);
        mma(a, b);
      }
      release();
    }
    if (!have_next && tile_next < total_tiles) tc_next = locate<BN>(tasks, ntasks, tile_next, uni);

    if constexpr (K3F) {
      // ---- K3f epilogue: +alpha acc and -alpha acc staged in shared memory (128B-swizzled boxes of
      // 16 columns x 128 rows), then one thread reduce-adds the right one into every output block
      // the leaf's W column touches.  Zero-filled rows / columns of a ragged tile add zeros.
      const unsigned stg_p = bars + 1024u, stg_n = stg_p + (unsigned)(BM * BN * 8);
      const bool issuer = cw == 0 && lane == 0;
      if (issuer) bulk_wait_read_all();  // the previous tile's reduces have read the staging tiles
      named_bar_sync(1, CONSUMERS * 32);
      const int cofs_k = (c == 0) ? 0 : (c == 1) ? 8 : (c == 2) ? 2 : 10;
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int row = wm + 16 * (i >> 1) + 2 * r + (i & 1);
#pragma unroll
        for (int jj = 0; jj < NI; ++jj) {
          const int col = wn + 16 * (jj >> 1) + 4 * (jj & 1) + cofs_k;  // even: a 16-byte pair
          const unsigned off = (unsigned)(col >> 4) * (unsigned)(BM * 128) + (unsigned)row * 128u +
                               ((((unsigned)(col & 15) >> 1) ^ (unsigned)(row & 7)) << 4);
          const double v0 = alpha * acc[i][jj][0], v1 = alpha * acc[i][jj][1];
          sts_f64x2(stg_p + off, v0, v1);
          sts_f64x2(stg_n + off, -v0, -v1);
        }
      }
      fence_proxy_async_shared();
      named_bar_sync(1, CONSUMERS * 32);
      if (issuer) {
        const int col_leaf = __ldg(&t.aux);
        const void* map = reinterpret_cast<const char*>(ka->maps) + 128 * __ldg(&t.node);
        const int nt = __ldg(&ka->count[col_leaf]);
        for (int q = 0; q < nt; ++q) {
          const K3fTarget tg = ka->targets[col_leaf * K3F_MAX_TARGETS + q];
          const unsigned src = tg.sign > 0 ? stg_p : stg_n;
#pragma unroll
          for (int b = 0; b < BN / 16; ++b)
            tma_reduce_add_2d(map, tg.col_off + tc.n0 + 16 * b, tg.row_off + tc.m0, src + (unsigned)(b * BM * 128));
        }
        bulk_commit();
      }
      continue;
    }
    const int cofs = (c == 0) ? 0 : (c == 1) ? 8 : (c == 2) ? 2 : 10;  // map0[2c]
    if constexpr (EPI) {
      // ---- staged epilogue: the warp writes alpha * acc into its sub-partition's staging slot and
      // its lanes hand the rows to the bulk-copy engine (cp.async.bulk shared -> global), so the
      // warp returns to the DMMAs of its next tile while the engine writes C.  The two warps of a
      // sub-partition (cw, cw + 4) take the slot in turn: named barrier 2 + q "slot staged and
      // read by the engine" (first -> second), 6 + q "second's copies have read it" (second ->
      // first, from the second tile on).  Tiles with beta != 0 keep the register epilogue below.
      // EPI = 2: one slot per warp (no hand-over; the warp only waits for its own previous copies)
      constexpr int STRIDE = epi_stride(BN, WGN);
      const int q = cw & 3;
      const bool second = EPI == 1 && cw >= CONSUMERS / 2;
      const unsigned slot = bars + 256u + (unsigned)(EPI == 2 ? cw : q) * (unsigned)epi_slot_bytes(BN, WGM, WGN);
      if (EPI == 2) {
        bulk_wait_read_all();
        __syncwarp();
      } else if (!second) {
        if (tile != (int)blockIdx.x) named_bar_sync(6 + q, 64);
      } else {
        if (tile != (int)blockIdx.x) {
          bulk_wait_read_all();
          __syncwarp();
          named_bar_arrive(6 + q, 64);
        }
        named_bar_sync(2 + q, 64);
      }
      const bool staged = beta == 0.0;
      if (staged) {
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int lr = 16 * (i >> 1) + 2 * r + (i & 1);
#pragma unroll
          for (int jj = 0; jj < NI; ++jj) {
            const int lc = 16 * (jj >> 1) + 4 * (jj & 1) + cofs;
            sts_f64x2(slot + (unsigned)(lr * STRIDE + lc * 8), alpha * acc[i][jj][0], alpha * acc[i][jj][1]);
          }
        }
        fence_proxy_async_shared();
        __syncwarp();
        const int gcol = tc.n0 + wn;
        const int nc = min(WTN, n - gcol);
        if (nc > 0) {
          for (int lr = lane; lr < WTM; lr += 32) {
            const int grow = tc.m0 + wm + lr;
            if (grow >= m) break;
            double* dst = C + (long long)grow * ldc + gcol;
            const unsigned src = slot + (unsigned)(lr * STRIDE);
            if (nc >= 2) bulk_store(dst, src, (unsigned)(nc & ~1) * 8u);
            if (nc & 1) dst[nc - 1] = lds64(src + (unsigned)(nc - 1) * 8u);
          }
        }
        bulk_commit();
      }
      if (EPI == 1 && !second) {
        if (staged) bulk_wait_read_all();
        __syncwarp();
        named_bar_arrive(2 + q, 64);
      }
      if (staged) continue;
    }
    // ---- epilogue: C = alpha * acc (+ beta * C), from registers ----
    // Interior warp tiles with beta = 0 (all but the ragged edge of a leaf) take a straight-line
    // form: one base pointer, compile-time offsets, no per-element range or beta branches.  ncu's
    // source page put 3.5 % of c5t's samples on the general form's ~700 instructions (BSSY / BRA
    // around every store), i.e. the tile boundary was issue-bound, not store-bound (DESIGN 6d).
#if !defined(FMM_GEMM_NOSTORE) && !defined(FMM_GEMM_NO_FAST_EPI)
    if (beta == 0.0 && tc.m0 + wm + WTM <= m && tc.n0 + wn + WTN <= n) {
      double* c0 = C + (long long)(tc.m0 + wm + 2 * r) * ldc + (tc.n0 + wn + cofs);
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        double* crow = c0 + (long long)(16 * (i >> 1) + (i & 1)) * ldc;
#pragma unroll
        for (int jj = 0; jj < NI; ++jj) {
          double2* p = reinterpret_cast<double2*>(crow + 16 * (jj >> 1) + 4 * (jj & 1));
          const double v0 = alpha * acc[i][jj][0], v1 = alpha * acc[i][jj][1];
#if FMM_GEMM_STG == 2
          __stcs(p, make_double2(v0, v1));
#elif FMM_GEMM_STG == 1
          st_global_v2(p, v0, v1);
#else
          *p = make_double2(v0, v1);
#endif
        }
      }
    } else
#endif
    {
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int row = tc.m0 + wm + 16 * (i >> 1) + 2 * r + (i & 1);
      if (row >= m) continue;
#ifdef FMM_GEMM_NOSTORE  // timing experiment: the epilogue's cost (stores only for an impossible value)
      if (acc[i][0][0] != 1.2345e300) continue;
#endif
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
#if FMM_GEMM_STG == 2
          __stcs(p, make_double2(v0, v1));
#elif FMM_GEMM_STG == 1
          st_global_v2(p, v0, v1);
#else
          *p = make_double2(v0, v1);
#endif
        } else if (col < n) {
          crow[col] = beta != 0.0 ? fma(beta, crow[col], v0) : v0;
        }
      }
    }
    }
    if constexpr (FUSED) {  // publish the stored tile (release) to the assembly jobs of its parent
      __threadfence();
      named_bar_sync(1, CONSUMERS * 32);
      if (cw == 0 && lane == 0) atomicAdd(&fa.ctr[2 + fa.np + __ldg(&t.node)], 1ull);
    }
  }
  if constexpr (FUSED) {
    for (;;) {
      const int idx = claim(&fa.ctr[1], lane);
      if (fa.njobs0 + idx >= fa.njobs) break;
      run_job(fa, fa.njobs0 + idx, lane, sp);
    }
  }
  if constexpr (K3F) {
    if (cw == 0 && lane == 0) bulk_wait_all();  // the last reduces complete before the CTA's smem goes
  }
  if constexpr (EPI) bulk_wait_all();  // the last tile's row copies, before the CTA's smem goes
}

}  // namespace fmm
