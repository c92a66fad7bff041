// Internal declarations of libfmm (not part of the C ABI).  Shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/fmm.h"
#include "fmm_device.cuh"

namespace fmm {

// ---- errors --------------------------------------------------------------------------------
struct Error : std::runtime_error {
  fmm_status_t code;
  Error(fmm_status_t c, const std::string& m) : std::runtime_error(m), code(c) {}
};
void set_last_error(const std::string& msg);

// Every extern "C" entry point wraps its body in these: no C++ exception crosses the ABI.
#define FMM_API_BEGIN try {
#define FMM_API_END                              \
  }                                              \
  catch (const ::fmm::Error& e) {                \
    ::fmm::set_last_error(e.what());             \
    return e.code;                               \
  }                                              \
  catch (const std::bad_alloc&) {                \
    ::fmm::set_last_error("host out of memory"); \
    return FMM_E_NO_MEMORY;                      \
  }                                              \
  catch (const std::exception& e) {              \
    ::fmm::set_last_error(e.what());             \
    return FMM_E_INVALID_ARG;                    \
  }
#define FMM_CUDA(x)                                                                              \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess)                                                                       \
      throw ::fmm::Error(FMM_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_) + " (" + \
                                         __FILE__ + ":" + std::to_string(__LINE__) + ")");      \
  } while (0)

// ---- exact rationals (coefficient storage, Brent check) ------------------------------------
struct Rat {
  __int128 n = 0, d = 1;  // d > 0, gcd(n, d) = 1
};
Rat rat_make(__int128 n, __int128 d);
Rat rat_add(Rat a, Rat b);
Rat rat_mul(Rat a, Rat b);
inline bool rat_is_zero(const Rat& a) { return a.n == 0; }
inline double rat_to_double(const Rat& a) { return (double)a.n / (double)a.d; }

}  // namespace fmm

// The algorithm object behind the opaque ABI handle.
struct fmm_alg_s {
  int M, K, N, R;
  std::vector<fmm::Rat> U, V, W;   // row-major MK x R, KN x R, MN x R
  std::vector<double> Ud, Vd, Wd;  // the same as doubles
};

namespace fmm {

// multi-GPU combine (fmm_dist.cpp): in-place NCCL sum-reduce of a contiguous C to `root`
void dist_reduce(void* comm, double* C, size_t count, int root, cudaStream_t stream);
void dist_reduce_slabs(void* comm, int nranks, double* C, long long outer, long long inner, cudaStream_t stream);
void dist_slab_range(long long outer, int nranks, int rank, long long* r0, long long* r1);
// grouped in-place NCCL reduces of row ranges [first, second) of a contiguous rows x inner C: each
// range to `root`, or (root = FMM_DIST_SLABS) each range's intersection with slab g to rank g
void dist_reduce_rows(void* comm, int nranks, double* C, long long rows, long long inner,
                      const std::vector<std::pair<long long, long long>>& ranges, int root, cudaStream_t stream);
// the peer-memory combine (fmm_p2p.cu)
void p2p_reduce_rows(const fmm_p2p* p, long long outer, long long r0, long long r1, long long inner, long long ld,
                     double* out, long long ldo, cudaStream_t s);
int p2p_nranks(const fmm_p2p* p);
int p2p_rank(const fmm_p2p* p);
int p2p_device(const fmm_p2p* p);
double* p2p_local(const fmm_p2p* p);
double* p2p_peer(const fmm_p2p* p, int g);  // rank g's buffer as mapped in this process
size_t p2p_bytes(const fmm_p2p* p);
// push mode: out = sum over g ascending of slot g (slot_elems apart) of this rank's buffer, rows x
// inner with leading dimension ld in each slot
void p2p_reduce_slots(const fmm_p2p* p, long long slot_elems, long long rows, long long inner, long long ld,
                      double* out, long long ldo, cudaStream_t s);
void* comm_handle(const fmm_comm* c);
int comm_nranks(const fmm_comm* c);
int comm_rank(const fmm_comm* c);
int comm_device(const fmm_comm* c);

fmm_alg* alg_transpose_prop1(const fmm_alg& a);  // Prop. 1: <N,K,M>
fmm_alg* alg_cycle_prop2(const fmm_alg& a);      // Prop. 2: <N,M,K>
void alg_validate_exact(const fmm_alg& a);        // throws FMM_E_NOT_EXACT

// ---- grouped DMMA GEMM (K2 / K4 / K5) -------------------------------------------------------
// GemmTask, FusedJob, FusedArgs: fmm_device.cuh (shared with the NVRTC-compiled fused kernel)
// Fill tiles_m/tiles_n/tile_begin; returns the total number of CTA tiles.
long long gemm_prepare(std::vector<GemmTask>& tasks, int bm = 128, int bn = 128);
bool gemm_tasks_aligned16(const std::vector<GemmTask>& tasks);
// Launch over a device copy of the prepared task list.
void gemm_launch(const GemmTask* d_tasks, int ntasks, long long total_tiles, bool aligned16,
                 cudaStream_t stream);
int gemm_tile_m();
int gemm_tile_n();
// TMA + warp-specialised variant (fmm_gemm_tma.cu): needs 16-byte aligned views, even lds.
bool gemm_tma_eligible(const std::vector<GemmTask>& tasks);
size_t gemm_tma_map_bytes();  // bytes of one tensor map (two per task: A then B)
void gemm_tma_maps(const std::vector<GemmTask>& tasks, void* out, int ks);  // ks: the launch's k-step (B box rows)
int gemm_choose_bk(const std::vector<GemmTask>& tasks);                      // 16, 32 or 48
// staged epilogue (bulk-copy stores) for a launch of tile width bn: 1 / 0; may lower *bk so the
// ring fits beside the staging slots
int gemm_choose_epi(const std::vector<GemmTask>& tasks, int bn, int* bk);
constexpr int BK_K3F = 16;  // the K3f leaf GEMM's k-step (its maps and smem; fmm_gemm_core.cuh BK)
// uniform_tm/tn: the common tile grid when every task has the same one (else 0, 0).
void gemm_tma_launch(const GemmTask* d_tasks, const void* d_maps, int ntasks, long long total_tiles, int bn, int bk,
                     int uniform_tm, int uniform_tn, cudaStream_t stream, int epi = 0);
// K3f leaf GEMM (128 x K3F_BN tiles; epilogue reduce-adds into the W targets through TMA): the
// tensor map of one parent output block (box 16 columns x 128 rows, 128B swizzle) and the launch.
void gemm_k3f_target_map(void* out, const double* ptr, long long rows, long long cols, long long ld);
void gemm_k3f_launch(const GemmTask* d_tasks, const void* d_maps, int ntasks, long long total_tiles, int uniform_tm,
                     int uniform_tn, const K3fArgs& ka, cudaStream_t stream);
// One-launch path for small one-level plans (fmm_small.cu, option small_fused): a term of an
// operand / output combination -- block index in the base case's grid (A: M x K, B: K x N) or the
// product index r (W), and its coefficient; per r (per output block k) the terms [off[r], off[r+1]).
struct SmallTerm {
  long long off;  // A / B terms: element offset of the block in the operand (rebuilt per execute's lds)
  double coef;
  int blk;
  int pad_;
};
constexpr int SMALL_MAX_R = 64, SMALL_MAX_UV = 160, SMALL_MAX_W = 256;  // R, MN <= 64; nnz(U), nnz(V), nnz(W)
struct SmallArgs {
  const double* A;
  const double* B;
  double* C;
  long long lda, ldb, ldc;
  int pm, pk, pn;  // leaf dimensions (P / M, Q / K, N / N_base: the plan requires exact division)
  int M, K, N, R;  // base case
  int tiles_m, tiles_n;
  // the term tables travel in the kernel parameters (constant bank: no global loads in the prologue)
  int u_off[SMALL_MAX_R + 1], v_off[SMALL_MAX_R + 1], w_off[SMALL_MAX_R + 1];
  SmallTerm u_terms[SMALL_MAX_UV], v_terms[SMALL_MAX_UV], w_terms[SMALL_MAX_W];
  double* Mbuf;    // R x tiles x 32 x 32 doubles
  unsigned* cnt;   // 2 per tile position (arrive, depart), zero between launches
  int kc, g;       // k-chunk depth (16, 32 or 64) and assembly group (small_config)
  int stage_max;   // doubles of one raw chunk buffer (the largest term counts)
  int nw;          // W terms (<= 256)
  int vec2;        // 1: every A / B view is 16-byte aligned (16-byte copies)
  int cluster;     // 1: the R CTAs of a tile are a cluster (C_k from the peers' shared memory)
  int prefetch;    // 1: the next chunk's copies are issued before the current chunk is used
  int coop;        // 1: the whole grid is resident; the R CTAs of a tile assemble it together
  int direct;      // 1: the classical product (<1,1,1;1>, L = 0): each CTA writes its tile to C
  int smem;        // dynamic shared memory bytes of the launch
};
int small_tile();  // the tile edge (32)
// chunk depth / assembly group for the largest per-product term counts; false: does not fit
bool small_config(int max_nu, int max_nv, int pk, int R, int* kc, int* g);
void small_launch(const SmallArgs& a, cudaStream_t stream);
bool small_cluster_ok(int R, int smem);  // the cluster variant fits (R <= 16, co-resident)
bool small_coop_ok(long long grid, int smem, int kc, int vec2);  // every CTA of the launch is co-resident
// TMA kernel configuration: consumer warp grid of a tile width, SM count, dynamic shared memory.
void gemm_bn_config(int bn, int* wgm, int* wgn);
int gemm_sm_count();
int gemm_bk();      // k-depth of a TMA ring stage (FMM_GEMM_BK of the nvcc build)
int gemm_stages();  // ring stages (FMM_GEMM_STAGES of the nvcc build)
int gemm_tma_smem_bytes(int bn);
int gemm_fused_smem_bytes(int bn, int ks, int bg_stage = 0);
int gemm_max_smem_bytes();  // the device's opt-in dynamic shared memory per block
// (tiles_m, tiles_n) shared by every task of a prepared list, or (0, 0).
void gemm_uniform_grid(const std::vector<GemmTask>& tasks, int* tm, int* tn);
// Thin products (one dimension <= skinny_limit()) on the CUDA cores (fmm_skinny.cu): ids index
// the task table; row tasks have m <= limit, column tasks n <= limit.
int skinny_limit();
void skinny_launch(const GemmTask* d_tasks, const int* d_row_ids, int nrow, int max_n, const int* d_col_ids, int ncol,
                   int max_m, cudaStream_t stream, int thin_r = 8, int thin_c = 8);  // thin_r / thin_c: the
                   // largest row-strip height / column-strip width of the launch
// Pick the TMA kernel's tile width (128 rows x bn columns) for a task list from a cost model of
// padded work, measured per-width efficiency and wave quantisation; FMM_GEMM_BN overrides.
int gemm_choose_bn(const std::vector<GemmTask>& tasks);

// ---- linear-combination (addition chain) kernels, generated and compiled with NVRTC --------
// One kernel computes, for every element position of a block, out_o = sum_i coef[o][i] * in_i.
struct LincombSpec {
  int nin = 0, nout = 0;
  std::vector<double> coef;  // nout x nin, row-major; chain order = ascending input index
  int strategy = FMM_ADD_STREAMING;
  int cse = 0;
  int vec = 2;  // doubles per thread access (2 = 16-byte vectors)
  int skip_null = 0;  // streaming: a null input pointer reads as zeros (a shard's absent leaf products)
};
struct LincombKernel;  // compiled function handle
// Per-node pointer table entry layout used by every generated kernel:
//   const double* in[nin]; double* out[nout]; long long ld_in; long long ld_out;
size_t lincomb_node_bytes(int nin, int nout);
std::shared_ptr<LincombKernel> lincomb_get(const LincombSpec& spec);
// Launch over `nodes` node entries (device table) for blocks of rows x cols elements.
void lincomb_launch(const LincombKernel& k, const void* d_nodes, int nnodes, long long rows, long long cols,
                    cudaStream_t stream);
// Statistics of the generated code (for fmm_plan_stats): additions per element, and per-element
// reads/writes of the kernel as launched.
struct LincombCost {
  double adds_per_elem;
  double reads_per_elem;   // elements read (inputs) per element position
  double writes_per_elem;  // elements written per element position
};
// Two recursion levels in one streaming pass (the last two levels collapsed).
// Formation (side 0 / 1): inputs are the rows^2 sub-sub-blocks x[i1][i2] (index i1 * rows + i2) of
// a grandparent block; for every level-(L-1) column r1 the intermediate T[r1][i2] = sum_i1 X[i1][r1]
// x[i1][i2] (or x[i1s][i2] unscaled for a singleton r1), then output (r1, r2) (index r1 * R + r2) =
// sum_i2 X[i2][r2] T[r1][i2] (or T[r1][i2s] unscaled for a singleton r2) when materialize[r1 R + r2].
// Assembly (side 2): inputs are the R^2 leaf products M[r1][r2]; M1[r1][k2] = sum_r2 X[k2][r2]
// M[r1][r2], output (k1, k2) (index k1 * rows + k2) = sum_r1 X[k1][r1] M1[r1][k2].  Every chain is
// ascending-index with first-term initialisation, i.e. the oracle's two levels exactly.
struct TwoLevelSpec {
  int side = 0;               // 0 = A formation, 1 = B formation, 2 = assembly
  int rows = 0, R = 0;        // rows of X (MK, KN or MN), rank
  std::vector<double> X;      // rows x R, row-major (U, V or W)
  std::vector<char> materialize;  // formation: R*R flags
  int vec = 2;
  int skip_null = 0;  // assembly: a null input pointer reads as zeros (a shard's absent leaf products)
};
std::shared_ptr<LincombKernel> twolevel_get(const TwoLevelSpec& spec);
LincombCost lincomb_cost(const LincombKernel& k);
int lincomb_steps(const LincombKernel& k);               // launches per lincomb_launch (pairwise: max chain length)
int lincomb_out_terms(const LincombKernel& k, int q);   // terms in output q's chain
void lincomb_cse_program(const LincombSpec& spec, std::vector<std::tuple<int, int, double>>* temps,
                         std::vector<std::vector<std::pair<int, double>>>* outs);
int lincomb_cse_temps(const LincombKernel& k);
std::string lincomb_source(const LincombKernel& k);

// The fused leaf-level kernel: the GEMM core (fmm_gemm_core.cuh) plus the plan's addition programs
// as straight-line device code (the same chains as the K1/K3 kernels of `progs`), compiled with
// NVRTC for one tile width and ring depth ks (16, 32, 48); cached by source.  bg: background mode
// (FMM_FUSED_BG: the producer warpgroup's spare warps run the jobs, every CTA runs leaf tiles).
struct FusedKernel;
std::shared_ptr<FusedKernel> fused_get(const std::vector<LincombSpec>& specs, int bn, int ks, bool bg);
std::string fused_generate(const std::vector<LincombSpec>& specs, int bn, int ks, bool bg);  // host only
int fused_bg_stage_bytes(const std::vector<LincombSpec>& specs);  // per producer warp (background mode)
std::vector<char> fused_compile(const std::string& source);                  // host only (NVRTC -> cubin)
const LincombSpec& lincomb_spec(const LincombKernel& k);
void fused_launch(const FusedKernel& k, const GemmTask* d_tasks, const void* d_maps, int ntasks, long long total_tiles,
                  int uniform_tm, int uniform_tn, const FusedArgs& fa, cudaStream_t stream);
std::string fused_source(const FusedKernel& k);

}  // namespace fmm
