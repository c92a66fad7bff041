// K2 (main path): the persistent, warp-specialised grouped FP64 GEMM fed by TMA
// (fmm_gemm_core.cuh holds the kernel body and its design notes), and its host side: tensor maps,
// the tile-width choice and the launches.  Used whenever every operand view is 16-byte aligned
// with even leading dimensions (what TMA requires); fmm_gemm.cu covers the rest.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "fmm_internal.h"
#include "fmm_gemm_core.cuh"

namespace fmm {

namespace {

template <int BN, int WGM, int WGN, int KS, int EPI>
__global__ void __launch_bounds__(THREADS, 1)
    grouped_dgemm_tma(const GemmTask* __restrict__ tasks, const CUtensorMap* __restrict__ maps, int ntasks,
                      int total_tiles, Uniform uni) {
  gemm_body<BN, WGM, WGN, false, false, KS, EPI>(tasks, maps, ntasks, total_tiles, uni, FusedArgs{});
}

// K3f: the leaf GEMM whose epilogue reduce-adds every tile into its W targets (tile 128 x 64)
__global__ void __launch_bounds__(THREADS, 1)
    grouped_dgemm_k3f(const GemmTask* __restrict__ tasks, const CUtensorMap* __restrict__ maps, int ntasks,
                      int total_tiles, Uniform uni, K3fArgs ka) {
  gemm_body<K3F_BN, 4, 2, false, true>(tasks, maps, ntasks, total_tiles, uni, FusedArgs{}, &ka);
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

void make_map(CUtensorMap* m, const double* ptr, long long rows, long long cols, long long ld, int box_cols, int box_rows);
}  // namespace

void gemm_k3f_target_map(void* out, const double* ptr, long long rows, long long cols, long long ld) {
  make_map(reinterpret_cast<CUtensorMap*>(out), ptr, rows, cols, ld, 16, BM);  // 16 columns x 128 rows
}

// the uniform tile grid of a launch and the magic numbers its tile map divides with
static Uniform make_uniform(int tm, int tn) {
  Uniform u{tm * tn, tm, tn};
  if (u.tiles > 0) {
    u.magic_tiles = 0xFFFFFFFFu / (unsigned)u.tiles;
    u.magic_span = 0xFFFFFFFFu / (unsigned)(GROUP_M * tn);
  }
  return u;
}


void gemm_k3f_launch(const GemmTask* d_tasks, const void* d_maps, int ntasks, long long total_tiles, int uniform_tm,
                     int uniform_tn, const K3fArgs& ka, cudaStream_t stream) {
  if (total_tiles <= 0 || ntasks <= 0) return;
  static std::atomic<unsigned long long> configured{0};
  int dev_ = 0;
  FMM_CUDA(cudaGetDevice(&dev_));
  const unsigned long long bit = 1ull << (dev_ & 63);
  const size_t smem = (size_t)k3f_smem_bytes(K3F_BN);
  if (!(configured.load() & bit)) {
    FMM_CUDA(cudaFuncSetAttribute(grouped_dgemm_k3f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured.fetch_or(bit);
  }
  const Uniform uni = make_uniform(uniform_tm, uniform_tn);
  const int grid = (int)std::min<long long>(total_tiles, gemm_sm_count());
  grouped_dgemm_k3f<<<grid, THREADS, smem, stream>>>(d_tasks, reinterpret_cast<const CUtensorMap*>(d_maps), ntasks,
                                                      (int)total_tiles, uni, ka);
  FMM_CUDA(cudaGetLastError());
}

namespace {
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

void gemm_tma_maps(const std::vector<GemmTask>& tasks, void* out, int ks) {
  auto* maps = reinterpret_cast<CUtensorMap*>(out);
  for (size_t i = 0; i < tasks.size(); ++i) {
    const GemmTask& t = tasks[i];
    make_map(&maps[2 * i], t.A, t.m, t.k, t.lda, 16, BM);      // A view: m rows x k cols, box 128 x 16
    make_map(&maps[2 * i + 1], t.B, t.k, t.n, t.ldb, 16, ks);  // B view: k rows x n cols, box ks x 16
  }
}

// Deeper stages mean fewer stage hand-overs per flop.  Measured on the round-2 kernel (leaf GEMM /
// DMMA peak, 16 / 32 / 48-deep): c2 (k = 2048) 0.980 / 0.987 / 0.987, c4 (k = 600) 0.927 / 0.930 /
// 0.933, c5 (k = 2000) 0.953 / 0.953 / 0.960, c3 (k = 450) 0.920 / 0.917 / 0.920, c5t (k = 400)
// 0.915 / 0.912 / 0.918: 48-deep stages (two of them) wherever k is not tiny
int gemm_choose_bk(const std::vector<GemmTask>& tasks) {
  if (const char* e = getenv("FMM_GEMM_BK_RUN")) {
    const int v = atoi(e);
    return v == 48 || v == 32 ? v : 16;
  }
  double fl = 0, f = 0;
  for (const auto& t : tasks) {
    const double w = (double)t.m * t.n * (double)t.k;
    f += w;
    if (t.k >= 96) fl += w;
  }
  return f > 0 && fl >= 0.5 * f ? 48 : 16;
}

template <int BN, int WGM, int WGN, int KS, int EPI>
static void launch_cfg(const GemmTask* d_tasks, const void* d_maps, int ntasks, long long total_tiles, int sms,
                       Uniform uni, cudaStream_t stream) {
  if constexpr (EPI && epi_ring_stages(KS, BN, WGM, WGN, EPI == 2 ? 8 : 4) < 2) {
    throw Error(FMM_E_INVALID_ARG, "staged epilogue: the ring does not fit beside the staging slots");
  } else {
    static std::atomic<unsigned long long> configured{0};  // bit d: attribute set on device d
    int dev_ = 0;
    FMM_CUDA(cudaGetDevice(&dev_));
    const unsigned long long bit = 1ull << (dev_ & 63);
    auto kern = grouped_dgemm_tma<BN, WGM, WGN, KS, EPI>;
    const size_t smem = (size_t)(EPI ? gemm_epi_smem_bytes(BN, KS, WGM, WGN, EPI == 2 ? 8 : 4) : gemm_smem_bytes(BN, KS));
    if (!(configured.load() & bit)) {
      FMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      configured.fetch_or(bit);
    }
    const int grid = (int)std::min<long long>(total_tiles, sms);
    kern<<<grid, THREADS, smem, stream>>>(d_tasks, reinterpret_cast<const CUtensorMap*>(d_maps), ntasks,
                                          (int)total_tiles, uni);
    FMM_CUDA(cudaGetLastError());
  }
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
  // relative DMMA efficiency of each tile width per useful flop, measured on c2's 2048^3 leaves
  // with the padding divided out (profiles/r2_leaf_gemm_study.jsonl, round-2 kernel): nearly flat,
  // so the padding decides
  static const int menu[] = {128, 112, 96, 80, 64};
  static const double eff[] = {1.00, 0.998, 0.996, 0.996, 0.993};
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

void gemm_bn_config(int bn, int* wgm, int* wgn) {
  switch (bn) {
    case 128: *wgm = 2, *wgn = 4; return;
    case 112: *wgm = 8, *wgn = 1; return;
    case 96: *wgm = 4, *wgn = 2; return;
    case 80: *wgm = 8, *wgn = 1; return;
    case 64: *wgm = 4, *wgn = 2; return;
    default: throw Error(FMM_E_INVALID_ARG, "unsupported GEMM tile width " + std::to_string(bn));
  }
}

int gemm_sm_count() { return sm_count(); }
static_assert(BK_K3F == BK, "the K3f maps and kernel agree on the k-step");
int gemm_bk() { return BK; }
int gemm_stages() { return GEMM_STAGES; }
int gemm_tma_smem_bytes(int bn) { return gemm_smem_bytes(bn, BK); }
int gemm_fused_smem_bytes(int bn, int ks, int bg_stage) { return fused_smem_bytes(bn, ks, bg_stage); }
int gemm_max_smem_bytes() {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
    cudaGetLastError();
    return 232448;  // sm_100
  }
  return v;
}

template <int KS, int EPI>
static void launch_ks(const GemmTask* d_tasks, const void* d_maps, int ntasks, long long total_tiles, int bn, int sms,
                      Uniform uni, cudaStream_t stream) {
  switch (bn) {
    case 128: launch_cfg<128, 2, 4, KS, EPI>(d_tasks, d_maps, ntasks, total_tiles, sms, uni, stream); break;
    case 112: launch_cfg<112, 8, 1, KS, EPI>(d_tasks, d_maps, ntasks, total_tiles, sms, uni, stream); break;
    case 96: launch_cfg<96, 4, 2, KS, EPI>(d_tasks, d_maps, ntasks, total_tiles, sms, uni, stream); break;
    case 80: launch_cfg<80, 8, 1, KS, EPI>(d_tasks, d_maps, ntasks, total_tiles, sms, uni, stream); break;
    case 64: launch_cfg<64, 4, 2, KS, EPI>(d_tasks, d_maps, ntasks, total_tiles, sms, uni, stream); break;
    default: throw Error(FMM_E_INVALID_ARG, "unsupported GEMM tile width " + std::to_string(bn));
  }
}

// Staged epilogue (gemm_body EPI = 1): whether a launch uses it, and the ring depth that leaves
// room for its staging slots (48-deep stages where two of them still fit, else 32, else 16).
// FMM_GEMM_EPI = 0 / 1 overrides the choice.
// a launch whose ring does not fit beside eight slots falls back to the four shared ones
static int gemm_choose_epi_fallback(int bn, int* bk);
static constexpr bool epi_fits(int bn, int ks, int slots) {
  return bn == 128 ? epi_ring_stages(ks, 128, 2, 4, slots) >= 2
         : bn == 112 ? epi_ring_stages(ks, 112, 8, 1, slots) >= 2
         : bn == 96  ? epi_ring_stages(ks, 96, 4, 2, slots) >= 2
         : bn == 80  ? epi_ring_stages(ks, 80, 8, 1, slots) >= 2
                     : epi_ring_stages(ks, 64, 4, 2, slots) >= 2;
}
int gemm_choose_epi(const std::vector<GemmTask>& tasks, int bn, int* bk) {
  int epi = 0;
  if (const char* e = getenv("FMM_GEMM_EPI")) epi = atoi(e);
  (void)tasks;
  if (epi != 1 && epi != 2) return 0;
  const int slots = epi == 2 ? 8 : 4;
  while (*bk > 16 && !epi_fits(bn, *bk, slots)) *bk = *bk == 48 ? 32 : 16;
  if (epi_fits(bn, *bk, slots)) return epi;
  if (epi == 2) return gemm_choose_epi_fallback(bn, bk);
  return 0;
}

static int gemm_choose_epi_fallback(int bn, int* bk) {
  while (*bk > 16 && !epi_fits(bn, *bk, 4)) *bk = *bk == 48 ? 32 : 16;
  return epi_fits(bn, *bk, 4) ? 1 : 0;
}

void gemm_tma_launch(const GemmTask* d_tasks, const void* d_maps, int ntasks, long long total_tiles, int bn, int bk,
                     int uniform_tm, int uniform_tn, cudaStream_t stream, int epi) {
  const Uniform uni = make_uniform(uniform_tm, uniform_tn);
  if (total_tiles <= 0 || ntasks <= 0) return;
#ifdef FMM_BG_PROBE
  {  // FMM_BG_BYTES: bytes the idle producer warps copy in the background (timing experiment)
    static double* buf = nullptr;
    static long long n = 0;
    const char* e = getenv("FMM_BG_BYTES");
    const long long want = e ? atoll(e) / 16 : 0;  // elements per src / dst half
    if (want > 0 && want != n) {
      if (buf) FMM_CUDA(cudaFree(buf));
      FMM_CUDA(cudaMalloc(&buf, (size_t)want * 16));
      FMM_CUDA(cudaMemset(buf, 0, (size_t)want * 16));
      n = want;
    }
    const double* src = buf;
    double* dst = buf ? buf + n : nullptr;
    const long long nn = want > 0 && total_tiles > 1000 ? n : 0;  // the leaf GEMM only, not tiny strips
    FMM_CUDA(cudaMemcpyToSymbolAsync(fmm_bg_src, &src, sizeof(src), 0, cudaMemcpyHostToDevice, stream));
    FMM_CUDA(cudaMemcpyToSymbolAsync(fmm_bg_dst, &dst, sizeof(dst), 0, cudaMemcpyHostToDevice, stream));
    FMM_CUDA(cudaMemcpyToSymbolAsync(fmm_bg_n, &nn, sizeof(nn), 0, cudaMemcpyHostToDevice, stream));
  }
#endif
  const int sms = sm_count();
  if (epi == 1) {
    if (bk == 48) launch_ks<48, 1>(d_tasks, d_maps, ntasks, total_tiles, bn, sms, uni, stream);
    else if (bk == 32) launch_ks<32, 1>(d_tasks, d_maps, ntasks, total_tiles, bn, sms, uni, stream);
    else if (bk == 16) launch_ks<16, 1>(d_tasks, d_maps, ntasks, total_tiles, bn, sms, uni, stream);
    else throw Error(FMM_E_INVALID_ARG, "unsupported GEMM k-step " + std::to_string(bk));
    return;
  }
  if (epi == 2) {
    if (bk == 48) launch_ks<48, 2>(d_tasks, d_maps, ntasks, total_tiles, bn, sms, uni, stream);
    else if (bk == 32) launch_ks<32, 2>(d_tasks, d_maps, ntasks, total_tiles, bn, sms, uni, stream);
    else if (bk == 16) launch_ks<16, 2>(d_tasks, d_maps, ntasks, total_tiles, bn, sms, uni, stream);
    else throw Error(FMM_E_INVALID_ARG, "unsupported GEMM k-step " + std::to_string(bk));
    return;
  }
  if (bk == 48) launch_ks<48, 0>(d_tasks, d_maps, ntasks, total_tiles, bn, sms, uni, stream);
  else if (bk == 32) launch_ks<32, 0>(d_tasks, d_maps, ntasks, total_tiles, bn, sms, uni, stream);
  else if (bk == 16) launch_ks<16, 0>(d_tasks, d_maps, ntasks, total_tiles, bn, sms, uni, stream);
  else throw Error(FMM_E_INVALID_ARG, "unsupported GEMM k-step " + std::to_string(bk));
}

}  // namespace fmm
