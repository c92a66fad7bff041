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
constexpr int BM = 128, BK = 16, STAGES = 6;
constexpr int CONSUMERS = 8, THREADS = 128 + CONSUMERS * 32;  // warpgroup 0 = producer, 1-2 = consumers
constexpr int A_BYTES = BM * BK * 8;   // 16 KB
constexpr size_t smem_bytes(int bn) { return (size_t)STAGES * (A_BYTES + BK * bn * 8) + 1024 /*align*/ + 256 /*barriers*/; }
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

// BN columns per CTA tile, consumer warps arranged WGM x WGN (WGM * WGN = 8); warp tile
// (128 / WGM) x (BN / WGN), both multiples of 16 so the fragment permutations apply.
template <int BN, int WGM, int WGN>
__global__ void __launch_bounds__(THREADS, 1)
    grouped_dgemm_tma(const GemmTask* __restrict__ tasks, const CUtensorMap* __restrict__ maps, int ntasks,
                      int total_tiles, Uniform uni) {
  static_assert(WGM * WGN == CONSUMERS, "8 consumer warps");
  constexpr int WTM = BM / WGM, WTN = BN / WGN;
  static_assert(WTM % 16 == 0 && WTN % 16 == 0, "warp tile must be a multiple of 16");
  constexpr int MI = WTM / 8, NI = WTN / 8;
  constexpr int B_BYTES_T = BK * BN * 8;  // BN/16 boxes of 16 x 16
  constexpr int STAGE_T = A_BYTES + B_BYTES_T;
  extern __shared__ unsigned char smem_raw[];
  const unsigned raw = smem_u32(smem_raw);
  const unsigned base = (raw + 1023u) & ~1023u;  // 1024-byte alignment for the 128B swizzle
  const unsigned bars = base + STAGES * STAGE_T;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

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
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == 0 && lane == 0) {
      int stage = 0;
      unsigned phase = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const TileCoord tc = locate<BN>(tasks, ntasks, tile, uni);
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
  for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
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

template <int BN, int WGM, int WGN>
static void launch_cfg(const GemmTask* d_tasks, const void* d_maps, int ntasks, long long total_tiles, int sms,
                       Uniform uni, cudaStream_t stream) {
  static bool configured = false;  // per process; one device per process (torchrun)
  auto kern = grouped_dgemm_tma<BN, WGM, WGN>;
  if (!configured) {
    FMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes(BN)));
    configured = true;
  }
  const int grid = (int)std::min<long long>(total_tiles, sms);
  kern<<<grid, THREADS, smem_bytes(BN), stream>>>(d_tasks, reinterpret_cast<const CUtensorMap*>(d_maps), ntasks,
                                                 (int)total_tiles, uni);
  FMM_CUDA(cudaGetLastError());
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

void gemm_tma_launch(const GemmTask* d_tasks, const void* d_maps, int ntasks, long long total_tiles, int bn,
                     int uniform_tm, int uniform_tn, cudaStream_t stream) {
  const Uniform uni{uniform_tm * uniform_tn, uniform_tm, uniform_tn};
  if (total_tiles <= 0 || ntasks <= 0) return;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    FMM_CUDA(cudaGetDevice(&dev));
    FMM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  switch (bn) {
    case 128: launch_cfg<128, 2, 4>(d_tasks, d_maps, ntasks, total_tiles, sms, uni, stream); break;
    case 112: launch_cfg<112, 8, 1>(d_tasks, d_maps, ntasks, total_tiles, sms, uni, stream); break;
    case 96: launch_cfg<96, 4, 2>(d_tasks, d_maps, ntasks, total_tiles, sms, uni, stream); break;
    case 80: launch_cfg<80, 8, 1>(d_tasks, d_maps, ntasks, total_tiles, sms, uni, stream); break;
    case 64: launch_cfg<64, 4, 2>(d_tasks, d_maps, ntasks, total_tiles, sms, uni, stream); break;
    default: throw Error(FMM_E_INVALID_ARG, "unsupported GEMM tile width " + std::to_string(bn));
  }
}

}  // namespace fmm
