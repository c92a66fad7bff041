// Types shared by the host library, the nvcc-compiled kernels and the NVRTC-compiled fused
// leaf-level kernel (this file is embedded verbatim into the NVRTC source: no includes here).
#pragma once

namespace fmm {

// One product C = alpha A B + beta C of a grouped GEMM launch (row-major views).
struct GemmTask {
  const double* A;
  const double* B;
  double* C;
  long long lda, ldb, ldc;
  int m, n, k;
  int tiles_m, tiles_n;
  int tile_begin;  // prefix sum of tiles over the task list
  int node;        // fused leaf-level / K3f launch: parent (level L-1) node index; -1 elsewhere
  int aux;         // K3f launch: the leaf's own column r_L of W (selects its output targets)
  double alpha, beta;
};

// K3f (the output step fused into the leaf GEMM's epilogue): each leaf tile is
// reduce-added by TMA (cp.reduce.async.bulk.tensor .add.f64) into the level-(L-1) output blocks
// its W column touches: for leaf column r, target q < count[r] is the parent sub-block at
// (row_off, col_off) with coefficient sign (+1 / -1) -- C_k += w_kr M_r.
constexpr int K3F_MAX_TARGETS = 16;
constexpr int K3F_BN = 64;  // tile width of the K3f leaf GEMM (its staging tiles must fit beside the ring)
struct K3fTarget {
  int row_off, col_off, sign, pad;
};
struct K3fArgs {
  const void* maps;          // one CUtensorMap per parent node (its output block), 64-byte aligned
  const int* count;          // [R]
  const K3fTarget* targets;  // [R][K3F_MAX_TARGETS]
};

// Uniform launches (every task has the same tile grid, e.g. all leaves of a level) map a tile to
// its task by division; others binary-search the tile prefix sums in the task table.
struct Uniform {
  int tiles, tiles_m, tiles_n;  // tiles == 0: not uniform
  // floor((2^32 - 1) / d) for d = tiles and d = (raster group height) * tiles_n: the tile map divides
  // by multiply-high plus one correction instead of the ~25-instruction emulated division (the
  // tile boundary of the leaf GEMM is issue-bound, DESIGN 6d).  0: divide.
  unsigned magic_tiles = 0, magic_span = 0;
};

// ---- fused leaf level (K1 level L + K2 + K3 level L in one persistent launch) ----------------
// A job is a row range of one parent node's formation (F: S_r / T_r of its children) or assembly
// (A: its C_k = sum_r w_kr M_r) through one addition program, i.e. one lincomb node table (the
// K1/K3 layout: in[nin], out[nout], ld_in, ld_out per node) and its generated chains.
constexpr int GEMM_THREADS = 384;   // producer warpgroup + 2 consumer warpgroups (addition CTAs: 12 workers)
constexpr int FUSED_MAX_PROGS = 3;  // formation A side, formation B side, assembly
// per warp, a shared-memory copy of the current job's node pointers (in[], out[], ld_in, ld_out):
// the generated code reads them from there instead of holding up to 64 pointers in registers
constexpr int FUSED_PTR_SLOT = 576;
constexpr int FUSED_PTR_BYTES = (GEMM_THREADS / 32) * FUSED_PTR_SLOT;
struct FusedJob {
  int prog, node;  // program, node-table entry
  int row0, nrows;
  int dep;         // parent index: F jobs signal ready[dep], A jobs wait for tiles_done[dep]
  int kind;        // 0 = formation (F), 1 = assembly (A)
};
struct FusedArgs {
  const char* node_tab[FUSED_MAX_PROGS];  // per program: node table
  int node_bytes[FUSED_MAX_PROGS];
  int cols[FUSED_MAX_PROGS];              // block width (elements) per program
  int vec2[FUSED_MAX_PROGS];              // 16-byte aligned views, even lds and cols
  const FusedJob* jobs;
  int njobs0, njobs;                      // phase-0 jobs [0, njobs0), phase-1 jobs [njobs0, njobs)
  unsigned long long* ctr;                // [0] claim0, [1] claim1, [2 + p] ready[p], [2 + np + p] tiles_done[p]
  const int* ready_target;                // [np]
  const int* tiles_target;                // [np]
  int np;
  int gemm_ctas;                          // CTAs [0, gemm_ctas) run leaf tiles, the rest are addition CTAs
};

}  // namespace fmm
