// Internal declarations of libfmm (not part of the C ABI).  Shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/fmm.h"

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

fmm_alg* alg_transpose_prop1(const fmm_alg& a);  // Prop. 1: <N,K,M>
void alg_validate_exact(const fmm_alg& a);        // throws FMM_E_NOT_EXACT

// ---- grouped DMMA GEMM (K2 / K4 / K5) -------------------------------------------------------
struct GemmTask {
  const double* A;
  const double* B;
  double* C;
  long long lda, ldb, ldc;
  int m, n, k;
  int tiles_m, tiles_n;
  int tile_begin;  // prefix sum of tiles over the task list
  int node;        // fused leaf-level launch: parent (level L-1) node index; -1 elsewhere
  double alpha, beta;
};
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
void gemm_tma_maps(const std::vector<GemmTask>& tasks, void* out);
// uniform_tm/tn: the common tile grid when every task has the same one (else 0, 0).
void gemm_tma_launch(const GemmTask* d_tasks, const void* d_maps, int ntasks, long long total_tiles, int bn,
                     int uniform_tm, int uniform_tn, cudaStream_t stream);
// ---- fused leaf level (K1 level L + K2 + K3 level L in one persistent launch) ----------------
// Addition programs run by an interpreter inside the GEMM kernel's spare warps.  A program is one
// lincomb node table (the K1/K3 format: in[nin], out[nout], ld_in, ld_out per node) plus its chains
// without CSE: for output o the terms [ostart[o], ostart[o+1]) of (in, coef), ascending input index.
// The programs live in a small blob (FusedProg headers, then per program short ostart[nout+1],
// short in[nterms], double coef[nterms]) that every CTA copies into shared memory at start.
struct FusedProg {
  long long node_off;  // byte offset of the node table from the launch-table base
  int ostart_off, in_off, coef_off;  // byte offsets inside the program blob
  int nin, nout, node_bytes;
  int rows, cols;
  int vec2;            // every view 16-byte aligned, even lds and cols: 16-byte / bulk-copy paths
  int seg;             // staged segment width in doubles (multiple of 64), 0 = direct loads only
};
struct FusedJob {
  int prog, node;  // program, node-table entry
  int row0, nrows;
  int dep;         // parent index: F jobs signal ready[dep], A jobs wait for tiles_done[dep]
  int kind;        // 0 = formation (F), 1 = assembly (A)
};
struct FusedArgs {
  const char* base;             // launch-table base (node tables)
  const char* blob;             // program blob (global copy)
  int blob_bytes, nprogs;
  const FusedJob* jobs;
  int njobs0, njobs;            // phase-0 jobs [0, njobs0), phase-1 jobs [njobs0, njobs)
  unsigned long long* ctr;      // [0] claim0, [1] claim1, [2 + p] ready[p], [2 + np + p] tiles_done[p]
  const int* ready_target;      // [np]
  const int* tiles_target;      // [np]
  int np;
  int gemm_ctas;                // CTAs [0, gemm_ctas) run leaf tiles, the rest are addition CTAs
};
constexpr int FUSED_ADD_SEG_BYTES = 9216;  // per staging buffer (two per addition warp)
constexpr int FUSED_PROG_BYTES = 6144;     // shared-memory program area
void gemm_fused_launch(const GemmTask* d_tasks, const void* d_maps, int ntasks, long long total_tiles, int bn,
                       int uniform_tm, int uniform_tn, const FusedArgs& fa, cudaStream_t stream);
// (tiles_m, tiles_n) shared by every task of a prepared list, or (0, 0).
void gemm_uniform_grid(const std::vector<GemmTask>& tasks, int* tm, int* tn);
// Thin products (one dimension <= skinny_limit()) on the CUDA cores (fmm_skinny.cu): ids index
// the task table; row tasks have m <= limit, column tasks n <= limit.
int skinny_limit();
void skinny_launch(const GemmTask* d_tasks, const int* d_row_ids, int nrow, int max_n, const int* d_col_ids, int ncol,
                   int max_m, cudaStream_t stream);
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
LincombCost lincomb_cost(const LincombKernel& k);
int lincomb_cse_temps(const LincombKernel& k);
std::string lincomb_source(const LincombKernel& k);

}  // namespace fmm
