// L2: the plan compiler and executor.
//
// A plan turns (algorithm, P x Q x N problem, L steps, options) into a fixed sequence of kernel
// launches over a breadth-first recursion tree (the paper's BFS scheme, Sec. 4.2, P:804-821,
// with every node of a level processed by ONE batched launch instead of one OpenMP task each):
//
//   for l = 1..L:   K1 formation, A side: S of every level-l node from its parent's blocks
//                   K1 formation, B side: T likewise                       (Sec. 3.2)
//   level L:        K2 grouped DMMA GEMM over all leaves: M = alpha * S * T
//   for l = L..1:   K3 assembly: parent C_k = sum_r w_kr M_r
//                   K4 peel strips of the level-(l-1) nodes (grouped GEMM)
//
// Views: every operand is (pointer, leading dimension, scalar sigma).  A column of U or V with a
// single nonzero is not formed: the child view aliases the parent block and its coefficient is
// piped into sigma, which reaches the leaf GEMM as alpha.
// Peeling: core P' = M floor(P/M) etc. at every level; strips per SPEC S:287-295 (R7).
// Column-major: Prop. 1 transpose, the problem becomes N x Q x P with A and B swapped.
// Sharding: HYBRID arithmetic over GPUs: the first R^L - (R^L mod G) leaves are split
// evenly and contiguously, the remaining R^L mod G leaves are split by rows over all G.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing unless a tool is attached

#include <algorithm>
#include <array>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "fmm_internal.h"

using namespace fmm;

namespace {

struct View {
  double* ptr = nullptr;
  long long ld = 0;
  double sigma = 1.0;
};

struct Dims {
  long long P, Q, N;     // node problem at this level: (P x Q) * (Q x N)
  long long P1, Q1, N1;  // divisible core (only meaningful below the last level)
};
using PlanDims = Dims;

struct Launch {
  enum Kind { FORM_A, FORM_B, GEMM, ASSEMBLE, STRIPS, SKINNY, FUSED, REDUCE /* no kernel: reduce_rows only */,
              ZERO /* K3f: zero the level-(L-1) output blocks (cudaMemset2DAsync per block) */,
              SMALL /* small_fused: the whole one-level step as one launch (fmm_small.cu) */ } kind;
  int level = 0;
  size_t table_off = 0;  // byte offset in the device table buffer
  int count = 0;         // nodes / tasks
  long long rows = 0, cols = 0;
  std::shared_ptr<LincombKernel> kern;
  long long tiles = 0;
  bool aligned16 = true;
  bool tma = false;          // GEMM launches: TMA warp-specialised kernel
  int bn = 128;              // GEMM launches: CTA tile width
  int bk = 16;               // GEMM launches: k-depth of a TMA ring stage (16, 32 or 48)
  int epi = 0;               // GEMM launches: staged epilogue (bulk-copy stores of C)
  int uni_tm = 0, uni_tn = 0;  // GEMM launches: common tile grid of all tasks (0 = mixed)
  size_t ids_off = 0;        // SKINNY: int ids (row tasks then column tasks)
  int nrow = 0, ncol = 0, max_n = 0, max_m = 0;
  int thin_r = 0, thin_c = 0;  // SKINNY: largest row-strip height / column-strip width
  size_t maps_off = 0;       // byte offset of the tensor maps (2 per task)
  double elem_reads = 0, elem_writes = 0, elem_adds = 0;  // totals over the launch (elements)
  double flops = 0, gemm_bytes = 0;
  std::vector<int> node_ids;  // FORM / ASSEMBLE: parent node index of every table entry
  int nin = 0, nout = 0;      // ASSEMBLE: inputs / outputs per table entry
  bool k3f = false;           // GEMM: the K3f leaf GEMM (epilogue reduce-adds into the W targets)
  SmallArgs small{};          // SMALL: the launch's arguments (term tables included)
  size_t k3f_maps_off = 0, k3f_count_off = 0, k3f_targets_off = 0;  // GEMM k3f: its device tables
  std::vector<std::array<long long, 4>> zero_blocks;  // ZERO: (host pointer bits, ld, rows, cols)
  // NCCL distributed plans with dist_chunks: rows [first, second) of C (plan orientation) to reduce
  // on the communication stream once this launch is done (a chunk of the assembly that writes C)
  std::vector<std::pair<long long, long long>> reduce_rows;
  // FUSED: byte offsets of the program / job / target tables, and their sizes
  size_t jobs_off = 0, targets_off = 0;
  int njobs0 = 0, njobs = 0, np = 0, nprogs = 0;
  int gemm_ctas = 0;  // FUSED: CTAs running leaf tiles (the rest of the grid are addition CTAs)
  size_t prog_node_off[FUSED_MAX_PROGS] = {};
  int prog_node_bytes[FUSED_MAX_PROGS] = {}, prog_cols[FUSED_MAX_PROGS] = {}, prog_vec2[FUSED_MAX_PROGS] = {};
  std::shared_ptr<FusedKernel> fk;
};

long long round_up(long long x, long long m) { return (x + m - 1) / m * m; }
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

struct fmm_plan_s {
  int device = 0;
  void* dist_comm = nullptr;  // distributed plan: NCCL communicator (not owned) and root
  int dist_root = 0;
  bool dist_chunked = false;  // the last build split the C-writing assembly into reduced row chunks
  cudaStream_t s_comm = nullptr;     // NCCL chunk reduces run here, overlapping the next chunk
  std::vector<cudaEvent_t> ev_chunk;  // one per chunk launch, and the end of the comm stream's work
  fmm_p2p* p2p = nullptr;     // peer-memory distributed plan (fmm_plan_create_p2p): partial buffer owner
  fmm_barrier_fn barrier = nullptr;
  void* barrier_ctx = nullptr;
  fmm_plan_options opt{};
  bool colmajor = false;
  std::unique_ptr<fmm_alg> alg_t;  // Prop. 1 transpose (column-major plans)
  const fmm_alg* alg = nullptr;     // the algorithm run (row-major orientation)
  long long P = 0, Q = 0, N = 0;    // row-major problem dims after the transpose
  long long userP = 0, userQ = 0, userN = 0;
  int L = 0;
  int R = 0;
  std::vector<Dims> dims;  // levels 0..L
  std::vector<long long> nodes_at;  // R^l

  // columns of U / V: formed (nnz != 1) or singleton (block index, coefficient)
  std::vector<int> formU, formV;             // formed column list (order = kernel output order)
  std::vector<int> idxU, idxV;               // for each r: output slot if formed, else -1
  std::vector<int> singU, singV;             // for each r: block index if singleton
  std::vector<double> coefU, coefV;          // for each r: singleton coefficient

  // sharding
  long long leaves = 1;
  std::vector<long long> leaf_r0, leaf_r1;   // active row range of each leaf (r0 == r1: inactive)
  std::vector<std::vector<char>> needed;     // [level][node]
  std::vector<std::vector<char>> strip_owner;// [level][node]

  // workspace
  double* ws = nullptr;
  size_t ws_bytes = 0;
  std::vector<long long> ldS, ldT, ldM;
  std::vector<std::vector<long long>> offS, offT, offM;  // element offsets in ws, -1 = none
  std::vector<long long> offZero;                        // per level: zero M block (shared)

  bool use_tma = true;  // FMM_NO_TMA=1 forces the cp.async GEMM (diagnostics)
  bool fuse = true;     // fuse_leaf_level option (FMM_NO_FUSE=1 overrides)
  bool fuse_bg = false;  // fuse_leaf_level = 2: the jobs run in the GEMM CTAs' spare warps (FMM_FUSE_BG=1)
  bool collapse = false;  // the last two levels' formation / assembly in one pass each (sec. 6c)
  bool collapse_asm = false;  // the last two levels' assembly in one pass (with collapse, or the wide
                              // warp-per-column kernel for base cases with MN up to 16, sec. 6g)
  bool k3f = false;       // fuse_output: the level-L output step in the leaf GEMM's epilogue (K3f)
  bool tiled_peel = false;  // R7c: the last split's rows were peeled to 128-row-aligned leaves
  bool small = false;       // small_fused: one launch for the whole one-level step (sec. 6h)
  double* small_M = nullptr;     // its leaf-product tiles (R x tiles x 32 x 32)
  unsigned* small_cnt = nullptr;  // its per-tile completion counters
  unsigned long long* d_ctr = nullptr;  // fused launch counters: claim0, claim1, ready[np], tiles[np]
  size_t ctr_bytes = 0;
  // kernels (vec 2 / vec 1 variants created lazily)
  std::shared_ptr<LincombKernel> kU[3], kV[3], kW[3];

  // launch tables: `launches`/`h_tab` are the scratch of the last build; two device slots cache
  // the tables of the two most recent (A, B, C, ld) sets (the pipelined host path alternates two
  // staging buffer sets)
  std::vector<Launch> launches;
  std::vector<char> h_tab;
  char* h_pinned = nullptr;
  size_t tab_bytes = 0;
  struct Slot {
    char* d_tab = nullptr;
    bool valid = false;
    const double* A = nullptr;
    const double* B = nullptr;
    double* C = nullptr;
    long long lda = -1, ldb = -1, ldc = -1;
    std::vector<Launch> launches;
    unsigned long long used = 0;
    int runs = 0;                     // executes served by this slot
    cudaGraphExec_t gexec = nullptr;  // its launch sequence as a CUDA graph (cuda_graphs option)
  } slot[2];
  cudaStream_t s_cap = nullptr;  // private stream the graphs are captured on
  unsigned long long use_clock = 0;
  cudaEvent_t upload_done = nullptr;
  cudaEvent_t ev[8] = {};
  // fmm_execute_timed: an event after every launch, and the phase of each launch (0 formation,
  // 1 leaf products, 2 assembly, 3 peel strips, 4 combine)
  bool profile_launches = false;
  std::vector<cudaEvent_t> ev_l;
  std::vector<int> ev_l_phase;
  std::vector<int> ev_l_kind, ev_l_level;  // the launch behind each event (kind, recursion level)

  // host-execute staging: two buffer sets, copy-in / copy-out streams, ordering events
  double *sA[2] = {nullptr, nullptr}, *sB[2] = {nullptr, nullptr}, *sC[2] = {nullptr, nullptr};
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev_in[2] = {}, ev_comp[2] = {}, ev_out[2] = {};
  unsigned long long host_iter = 0;

  ~fmm_plan_s() {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    if (upload_done) cudaEventSynchronize(upload_done);
    cudaDeviceSynchronize();
    if (ws) cudaFree(ws);
    if (scratch) cudaFree(scratch);
    if (d_ctr) cudaFree(d_ctr);
    if (small_M) cudaFree(small_M);
    if (small_cnt) cudaFree(small_cnt);
    for (auto& sl : slot) {
      if (sl.d_tab) cudaFree(sl.d_tab);
      if (sl.gexec) cudaGraphExecDestroy(sl.gexec);
    }
    if (s_cap) cudaStreamDestroy(s_cap);
    if (s_comm) cudaStreamDestroy(s_comm);
    for (auto& e : ev_chunk)
      if (e) cudaEventDestroy(e);
    if (h_pinned) cudaFreeHost(h_pinned);
    for (int b = 0; b < 2; ++b) {
      if (sA[b]) cudaFree(sA[b]);
      if (sB[b]) cudaFree(sB[b]);
      if (sC[b]) cudaFree(sC[b]);
      for (cudaEvent_t e : {ev_in[b], ev_comp[b], ev_out[b]})
        if (e) cudaEventDestroy(e);
    }
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
    if (upload_done) cudaEventDestroy(upload_done);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : ev_l)
      if (e) cudaEventDestroy(e);
    cudaSetDevice(cur);
  }

  std::shared_ptr<LincombKernel> kernel(int side, int vec) {
    auto* slot = side == 0 ? kU : side == 1 ? kV : kW;
    if (slot[vec]) return slot[vec];
    slot[vec] = lincomb_get(spec_for(side, vec));
    return slot[vec];
  }
  // a sharded streaming plan points its assembly tables at null for the leaf products it does not
  // own (instead of a zero block): the kernels read them as zeros without the HBM traffic
  bool skip_absent() const { return opt.shard_count > 1 && opt.strategy == FMM_ADD_STREAMING && !fuse; }
  LincombSpec spec_for(int side, int vec) const {
    LincombSpec s;
    s.strategy = opt.strategy;
    s.cse = opt.cse;
    s.vec = vec;
    s.skip_null = side == 2 && skip_absent();
    const int M = alg->M, K = alg->K, Nb = alg->N;
    if (side == 0 || side == 1) {
      const int rows = side == 0 ? M * K : K * Nb;
      const auto& X = side == 0 ? alg->Ud : alg->Vd;
      const auto& form = side == 0 ? formU : formV;
      s.nin = rows;
      s.nout = (int)form.size();
      s.coef.assign((size_t)s.nin * s.nout, 0.0);
      for (int o = 0; o < s.nout; ++o)
        for (int i = 0; i < rows; ++i) s.coef[(size_t)o * rows + i] = X[(size_t)i * R + form[o]];
    } else {
      s.nin = R;
      s.nout = M * Nb;
      s.coef.assign((size_t)s.nin * s.nout, 0.0);
      for (int k = 0; k < M * Nb; ++k)
        for (int r = 0; r < R; ++r) s.coef[(size_t)k * R + r] = alg->Wd[(size_t)k * R + r];
    }
    return s;
  }

  long long node_first_leaf(int l, long long z) const {
    long long f = z;
    for (int q = l; q < L; ++q) f *= R;
    return f;
  }
  long long node_leaf_span_from(int l) const {  // level-l nodes under one level-1 node
    long long f = 1;
    for (int q = 1; q < l; ++q) f *= R;
    return f;
  }
  long long node_leaf_span(int l) const {
    long long f = 1;
    for (int q = l; q < L; ++q) f *= R;
    return f;
  }

  void setup_sharding() {
    const long long G = std::max(1, opt.shard_count), g = opt.shard_rank;
    leaves = nodes_at[L];
    const long long dfs = leaves % G, bfs = leaves - dfs;
    const long long per = bfs / G;
    std::vector<int64_t> r0(leaves), r1(leaves);
    // top-level ownership (shard_mode 1): rank of top-level product r1 (contiguous balanced ranges)
    auto top_owner = [&](long long r) {
      const long long base = R / G, extra = R % G;
      const long long cut = extra * (base + 1);
      return r < cut ? r / (base + 1) : extra + (base > 0 ? (r - cut) / base : 0);
    };
    if (opt.shard_mode == 1 && L >= 1) {
      const long long span = node_leaf_span(1);  // leaves under one top-level product
      for (long long z = 0; z < leaves; ++z) {
        const bool own = top_owner(z / span) == g;
        r0[z] = 0;
        r1[z] = own ? dims[L].P : 0;
      }
    } else if (fmm_shard_leaf_rows(leaves, dims[L].P, G, g, r0.data(), r1.data()) != FMM_OK) {
      throw Error(FMM_E_INVALID_ARG, "bad shard arguments");
    }
    leaf_r0.assign(r0.begin(), r0.end());
    leaf_r1.assign(r1.begin(), r1.end());
    needed.assign(L + 1, {});
    strip_owner.assign(L + 1, {});
    for (int l = 0; l <= L; ++l) {
      needed[l].assign(nodes_at[l], 0);
      strip_owner[l].assign(nodes_at[l], 0);
    }
    for (long long z = 0; z < leaves; ++z)
      if (leaf_r1[z] > leaf_r0[z]) needed[L][z] = 1;
    // strips of a node: computed by the rank owning its first leaf (rank 0 for remainder leaves)
    for (int l = 0; l < L; ++l) {
      const bool has_strips = dims[l].P1 < dims[l].P || dims[l].Q1 < dims[l].Q || dims[l].N1 < dims[l].N;
      if (!has_strips) continue;
      for (long long z = 0; z < nodes_at[l]; ++z) {
        const long long f = node_first_leaf(l, z);
        long long owner = f < bfs ? (per > 0 ? f / per : 0) : 0;
        if (opt.shard_mode == 1) owner = l == 0 ? 0 : top_owner(z / node_leaf_span_from(l));
        if (owner == g) strip_owner[l][z] = 1, needed[l][z] = 1;
      }
    }
    for (int l = L; l >= 1; --l)
      for (long long z = 0; z < nodes_at[l]; ++z)
        if (needed[l][z]) needed[l - 1][z / R] = 1;
    needed[0][0] = 1;  // the root always writes C (zeros if this shard owns nothing)
  }

  void setup_workspace() {
    ldS.assign(L + 1, 0);
    ldT.assign(L + 1, 0);
    ldM.assign(L + 1, 0);
    offS.assign(L + 1, {});
    offT.assign(L + 1, {});
    offM.assign(L + 1, {});
    offZero.assign(L + 1, -1);
    long long total = 0;
    auto take = [&](long long elems) {
      const long long o = total;
      total += round_up(elems, 32);  // 256-byte aligned blocks
      return o;
    };
    for (int l = 1; l <= L; ++l) {
      const Dims& d = dims[l];
      ldS[l] = round_up(d.Q, 16);
      ldT[l] = round_up(d.N, 16);
      ldM[l] = round_up(d.N, 16);
      offS[l].assign(nodes_at[l], -1);
      offT[l].assign(nodes_at[l], -1);
      offM[l].assign(nodes_at[l], -1);
      bool any_unneeded = false;
      // collapsed formation: S_r, T_r of level L-1 never materialised (sec. 6c); M_r of level L-1
      // only if its assembly is not collapsed too
      if (collapse && collapse_asm && l == L - 1) continue;
      const bool noM = collapse_asm && l == L - 1;  // the collapsed assembly never writes M at L-1
      const bool noST = collapse && l == L - 1;
      for (long long z = 0; z < nodes_at[l]; ++z) {
        const int r = (int)(z % R);
        if (!needed[l][z]) {
          any_unneeded = true;
          continue;
        }
        const int r1 = (int)((z / R) % R);
        // collapsed leaves: materialised unless both levels' columns are singletons (then an alias)
        const bool formA = collapse && l == L ? (idxU[r] >= 0 || idxU[r1] >= 0) : idxU[r] >= 0;
        const bool formB = collapse && l == L ? (idxV[r] >= 0 || idxV[r1] >= 0) : idxV[r] >= 0;
        if (formA && !noST) offS[l][z] = take(d.P * ldS[l]);
        if (formB && !noST) offT[l][z] = take(d.Q * ldT[l]);
        if (!noM) offM[l][z] = take(d.P * ldM[l]);
      }
      if (any_unneeded && !noM) offZero[l] = take(d.P * ldM[l]);
    }
    ws_bytes = (size_t)total * sizeof(double);
    if (opt.workspace_limit_bytes && ws_bytes > opt.workspace_limit_bytes)
      throw Error(FMM_E_NO_MEMORY, "plan needs " + std::to_string(ws_bytes) + " workspace bytes (all S_r, T_r, M_r of " +
                                       std::to_string(L) + " BFS levels resident, R/(MN) x the output per step, P:820) > limit " +
                                       std::to_string(opt.workspace_limit_bytes));
    if (ws_bytes) {
      cudaError_t e = cudaMalloc(&ws, ws_bytes);
      if (e != cudaSuccess) {
        cudaGetLastError();
        ws = nullptr;
        throw Error(FMM_E_NO_MEMORY, "cudaMalloc of " + std::to_string(ws_bytes) + " workspace bytes failed");
      }
      // zero blocks of partially-owned leaves and shared zero blocks must read as zeros
      FMM_CUDA(cudaMemset(ws, 0, ws_bytes));
    }
  }

  // memory-CSE temporaries (write-once / pairwise with CSE): an arena laid out by
  // every build in the same order, allocated after the dry build
  double* scratch = nullptr;
  size_t scratch_elems = 0, scratch_used = 0;
  double* scratch_take(long long elems) {
    const size_t off = scratch_used;
    scratch_used += (size_t)round_up(elems, 32);
    return scratch ? scratch + off : reinterpret_cast<double*>((uintptr_t)0x400000 + off * 8);  // dry build
  }
  bool emit_mcse(Launch::Kind kind, int level, int side, const std::vector<char>& tab, int nin, int nout, int count,
                 long long rows, long long cols, bool aligned, const std::vector<int>& node_ids);

  View opA(int l, long long z, const View& root) const;
  View opB(int l, long long z, const View& root) const;

  // the execute arguments of the build in progress (row-major orientation)
  const double *cur_A = nullptr, *cur_B = nullptr;
  double* cur_C = nullptr;
  long long cur_lda = 0, cur_ldb = 0, cur_ldc = 0;
  size_t push_tab(const void* p, size_t n) {
    const size_t off = h_tab.size();
    h_tab.resize(align256(off + n));
    if (p && n) std::memcpy(h_tab.data() + off, p, n);
    return off;
  }
  // output block of node z at level l (C itself at the root; a shared zero block for nodes this
  // shard does not compute)
  View out_view(int l, long long z) const {
    if (l == 0) return View{cur_C, cur_ldc, 1.0};
    if (offM[l][z] >= 0) return View{ws + offM[l][z], ldM[l], 1.0};
    return View{offZero[l] >= 0 ? ws + offZero[l] : nullptr, ldM[l], 1.0};
  }

  // Build every launch and its table for the given execute arguments (row-major orientation).
  void build(const double* A, long long lda, const double* B, long long ldb, double* C, long long ldc, bool lazy_kernels);
  // Replace the level-L formation, leaf GEMM and level-L assembly launches by one fused launch.
  void fuse_leaf_level(bool lazy_kernels);
  // Collapsed levels L-1 and L (sec. 6c): one formation launch per side and one assembly launch
  // over the level-(L-2) nodes.
  void emit_two_level_formation(bool lazy_kernels);
  void emit_two_level_assembly(bool lazy_kernels);
  // NCCL distributed plans: split the assembly launch that writes C into dist_chunks row chunks,
  // each followed by the reduce of its rows of C (run() issues it on s_comm)
  void chunk_final_assembly();
  // K3f: zero the level-(L-1) outputs, then the leaf GEMM whose epilogue reduce-adds every tile
  // into its W targets (replaces the level-L assembly)
  void emit_k3f(std::vector<GemmTask>& tasks, bool lazy_kernels);
  // small_fused: the one launch of a small one-level plan and its term tables
  void emit_small();
};

View fmm_plan_s::opA(int l, long long z, const View& root) const {
  if (l == 0) return root;
  const int r = (int)(z % R);
  if (collapse && l == L) {  // leaf of two collapsed levels: relative to the grandparent
    const int r1 = (int)((z / R) % R);
    const View g = opA(L - 2, z / R / R, root);
    const double sig = g.sigma * (idxU[r1] < 0 ? coefU[r1] : 1.0) * (idxU[r] < 0 ? coefU[r] : 1.0);
    if (idxU[r1] >= 0 || idxU[r] >= 0) return View{offS[l][z] >= 0 ? ws + offS[l][z] : nullptr, ldS[l], sig};
    const int i1 = singU[r1], i2 = singU[r];
    const Dims &d1 = dims[L - 1], &d2 = dims[L];
    const long long off = (i1 / alg->K) * d1.P * g.ld + (i1 % alg->K) * d1.Q + (i2 / alg->K) * d2.P * g.ld + (i2 % alg->K) * d2.Q;
    return View{g.ptr ? g.ptr + off : nullptr, g.ld, sig};
  }
  const View par = opA(l - 1, z / R, root);
  if (idxU[r] >= 0) return View{offS[l][z] >= 0 ? ws + offS[l][z] : nullptr, ldS[l], par.sigma};
  const int i = singU[r];
  const Dims& d = dims[l];
  return View{par.ptr ? par.ptr + (i / alg->K) * d.P * par.ld + (i % alg->K) * d.Q : nullptr, par.ld,
              par.sigma * coefU[r]};
}

View fmm_plan_s::opB(int l, long long z, const View& root) const {
  if (l == 0) return root;
  const int r = (int)(z % R);
  if (collapse && l == L) {
    const int r1 = (int)((z / R) % R);
    const View g = opB(L - 2, z / R / R, root);
    const double sig = g.sigma * (idxV[r1] < 0 ? coefV[r1] : 1.0) * (idxV[r] < 0 ? coefV[r] : 1.0);
    if (idxV[r1] >= 0 || idxV[r] >= 0) return View{offT[l][z] >= 0 ? ws + offT[l][z] : nullptr, ldT[l], sig};
    const int j1 = singV[r1], j2 = singV[r];
    const Dims &d1 = dims[L - 1], &d2 = dims[L];
    const long long off = (j1 / alg->N) * d1.Q * g.ld + (j1 % alg->N) * d1.N + (j2 / alg->N) * d2.Q * g.ld + (j2 % alg->N) * d2.N;
    return View{g.ptr ? g.ptr + off : nullptr, g.ld, sig};
  }
  const View par = opB(l - 1, z / R, root);
  if (idxV[r] >= 0) return View{offT[l][z] >= 0 ? ws + offT[l][z] : nullptr, ldT[l], par.sigma};
  const int j = singV[r];
  const Dims& d = dims[l];
  return View{par.ptr ? par.ptr + (j / alg->N) * d.Q * par.ld + (j % alg->N) * d.N : nullptr, par.ld,
              par.sigma * coefV[r]};
}

static bool al16(const void* p);
// small_fused (sec. 6h): one SMALL launch; its term tables list, per product r, the nonzero
// u_ir (v_jr) with their block index in A's M x K (B's K x N) grid, and per output block k the
// nonzero w_kr in ascending r -- the orders of the separate kernels' chains without CSE
void fmm_plan_s::emit_small() {
  const fmm_alg* a = alg;
  // L = 0 (the classical product below the cutoff): the same kernel with the trivial base case
  // <1,1,1;1>, each CTA writing its tile of C directly
  const bool direct = L == 0;
  const int M = direct ? 1 : a->M, K = direct ? 1 : a->K, Nb = direct ? 1 : a->N, R = direct ? 1 : this->R;
  const std::vector<double> one{1.0};
  auto terms = [&](const std::vector<double>& X, int rows, bool by_r, std::vector<int>& off, std::vector<SmallTerm>& t) {
    const int outer = by_r ? R : rows, inner = by_r ? rows : R;
    off.assign(outer + 1, 0);
    for (int o = 0; o < outer; ++o) {
      for (int i = 0; i < inner; ++i) {
        const double c = by_r ? X[(size_t)i * R + o] : X[(size_t)o * R + i];
        if (c != 0.0) t.push_back(SmallTerm{0, c, i, 0});
      }
      off[o + 1] = (int)t.size();
    }
  };
  std::vector<int> uo, vo, wo;
  std::vector<SmallTerm> ut, vt, wt;
  terms(direct ? one : a->Ud, M * K, true, uo, ut);
  terms(direct ? one : a->Vd, K * Nb, true, vo, vt);
  terms(direct ? one : a->Wd, M * Nb, false, wo, wt);
  Launch ln;
  ln.kind = Launch::SMALL;
  ln.level = direct ? 0 : 1;
  const Dims& d = dims[direct ? 0 : 1];
  for (auto& tm : ut) tm.off = (tm.blk / K) * d.P * cur_lda + (tm.blk % K) * d.Q;
  for (auto& tm : vt) tm.off = (tm.blk / Nb) * d.Q * cur_ldb + (tm.blk % Nb) * d.N;
  const int T = small_tile();
  SmallArgs& sa = ln.small;
  std::copy(uo.begin(), uo.end(), sa.u_off);
  std::copy(vo.begin(), vo.end(), sa.v_off);
  std::copy(wo.begin(), wo.end(), sa.w_off);
  std::copy(ut.begin(), ut.end(), sa.u_terms);
  std::copy(vt.begin(), vt.end(), sa.v_terms);
  std::copy(wt.begin(), wt.end(), sa.w_terms);
  sa.A = cur_A, sa.B = cur_B, sa.C = cur_C;
  sa.lda = cur_lda, sa.ldb = cur_ldb, sa.ldc = cur_ldc;
  sa.pm = (int)d.P, sa.pk = (int)d.Q, sa.pn = (int)d.N;
  sa.M = M, sa.K = K, sa.N = Nb, sa.R = R;
  sa.tiles_m = (int)((d.P + T - 1) / T), sa.tiles_n = (int)((d.N + T - 1) / T);
  sa.Mbuf = small_M, sa.cnt = small_cnt;
  int max_nu = 0, max_nv = 0;
  for (int r = 0; r < R; ++r) max_nu = std::max(max_nu, uo[r + 1] - uo[r]), max_nv = std::max(max_nv, vo[r + 1] - vo[r]);
  if (!small_config(max_nu, max_nv, sa.pk, R, &sa.kc, &sa.g)) throw Error(FMM_E_UNSUPPORTED, "internal: small_fused config");
  sa.stage_max = max_nu * T * (sa.kc + 4) + max_nv * sa.kc * (T + 8);
  sa.smem = std::max({8 * (2 * sa.stage_max + T * (sa.kc + 4) + sa.kc * (T + 8)), 8 * R * sa.g, 3 * T * T * 8});
  sa.nw = (int)wt.size();
  sa.direct = direct ? 1 : 0;
  bool v2 = al16(cur_A) && al16(cur_B) && cur_lda % 2 == 0 && cur_ldb % 2 == 0;
  for (const auto& tm : ut) v2 = v2 && tm.off % 2 == 0;
  for (const auto& tm : vt) v2 = v2 && tm.off % 2 == 0;
  sa.vec2 = v2 ? 1 : 0;
  // the cluster variant (C_k over distributed shared memory) measured slower on c1 (26.7 against
  // 18.5 us per step): only on request (FMM_SMALL_CLUSTER=1)
  const char* cl = getenv("FMM_SMALL_CLUSTER");
  sa.cluster = !direct && cl && cl[0] == '1' && R >= M * Nb && small_cluster_ok(R, sa.smem);
  sa.prefetch = !(getenv("FMM_SMALL_PREFETCH") && getenv("FMM_SMALL_PREFETCH")[0] == '0');
  // the R CTAs of a tile assemble it together when the whole grid is resident (else the last one)
  sa.coop = !direct && !sa.cluster && small_coop_ok((long long)sa.tiles_m * sa.tiles_n * R, sa.smem, sa.kc, sa.vec2) && !(getenv("FMM_SMALL_COOP") && getenv("FMM_SMALL_COOP")[0] == '0');
  ln.count = R;
  ln.tiles = (long long)sa.tiles_m * sa.tiles_n * R;
  // work: the leaf products, the formation reads / adds and the assembly (as the separate kernels)
  ln.flops = 2.0 * R * d.P * (double)d.Q * d.N;
  ln.gemm_bytes = 8.0 * R * (d.P * d.Q + d.Q * d.N + d.P * d.N);
  ln.elem_reads = direct ? 0.0 : (double)ut.size() * d.P * d.Q + (double)vt.size() * d.Q * d.N + (double)wt.size() * d.P * d.N;
  ln.elem_writes = direct ? 0.0 : (double)M * Nb * d.P * d.N;
  ln.elem_adds = direct ? 0.0
                        : (double)(ut.size() - uo.size() + 1) * d.P * d.Q + (double)(vt.size() - vo.size() + 1) * d.Q * d.N +
                              (double)(wt.size() - M * Nb) * d.P * d.N;
  launches.push_back(ln);
}

static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

void fmm_plan_s::build(const double* A, long long lda, const double* B, long long ldb, double* C, long long ldc,
                       bool lazy_kernels) {
  launches.clear();
  h_tab.clear();
  scratch_used = 0;
  cur_A = A, cur_B = B, cur_C = C, cur_lda = lda, cur_ldb = ldb, cur_ldc = ldc;
  if (small) {  // the whole step as one launch (sec. 6h)
    emit_small();
    return;
  }
  const View rootA{const_cast<double*>(A), lda, 1.0}, rootB{const_cast<double*>(B), ldb, 1.0};
  const int M = alg->M, K = alg->K, Nb = alg->N;
  auto push = [&](const void* p, size_t n) {
    size_t off = h_tab.size();
    h_tab.resize(align256(off + n));
    if (p) std::memcpy(h_tab.data() + off, p, n);
    return off;
  };
  auto choose_tiles = [&](Launch& ln, std::vector<GemmTask>& tasks) {
    ln.tma = !lazy_kernels && use_tma && gemm_tma_eligible(tasks);
    ln.bn = ln.tma ? gemm_choose_bn(tasks) : 128;
    // (the fused leaf level reuses this launch's tensor maps and ring depth)
    ln.bk = ln.tma ? gemm_choose_bk(tasks) : 16;
    ln.epi = ln.tma ? gemm_choose_epi(tasks, ln.bn, &ln.bk) : 0;
    ln.tiles = gemm_prepare(tasks, 128, ln.bn);
    gemm_uniform_grid(tasks, &ln.uni_tm, &ln.uni_tn);
  };
  auto push_maps = [&](Launch& ln, const std::vector<GemmTask>& tasks) {
    if (lazy_kernels) {  // dry build: reserve the space the maps would need
      ln.maps_off = push(nullptr, 2 * gemm_tma_map_bytes() * tasks.size());
      return;
    }
    std::vector<char> maps(2 * gemm_tma_map_bytes() * tasks.size());
    if (ln.tma) gemm_tma_maps(tasks, maps.data(), ln.bk);
    ln.maps_off = push(maps.data(), maps.size());
  };
  // one grouped DMMA launch for the regular tasks, one CUDA-core launch for thin ones
  auto emit_gemm = [&](Launch::Kind kind, int level, std::vector<GemmTask>& all) {
    std::vector<GemmTask> reg, thin;
    for (const auto& t : all) {
      if (t.m <= 0 || t.n <= 0) continue;
      (std::min(t.m, t.n) <= skinny_limit() ? thin : reg).push_back(t);
    }
    if (!reg.empty()) {
      Launch ln;
      ln.kind = kind;
      ln.level = level;
      choose_tiles(ln, reg);
      ln.count = (int)reg.size();
      ln.aligned16 = gemm_tasks_aligned16(reg);
      for (auto& t : reg) {
        ln.flops += 2.0 * t.m * t.n * (double)t.k;
        ln.gemm_bytes += 8.0 * ((double)t.m * t.k + (double)t.k * t.n + (1.0 + (t.beta != 0.0)) * t.m * t.n);
      }
      ln.table_off = push(reg.data(), reg.size() * sizeof(GemmTask));
      push_maps(ln, reg);
      launches.push_back(ln);
    }
    if (!thin.empty()) {
      Launch ln;
      ln.kind = Launch::SKINNY;
      ln.level = level;
      ln.count = (int)thin.size();
      std::vector<int> rows, cols;
      for (int q = 0; q < (int)thin.size(); ++q) {
        const auto& t = thin[q];
        if (t.m <= skinny_limit()) rows.push_back(q), ln.max_n = std::max(ln.max_n, t.n), ln.thin_r = std::max(ln.thin_r, t.m);
        else cols.push_back(q), ln.max_m = std::max(ln.max_m, t.m), ln.thin_c = std::max(ln.thin_c, t.n);
        ln.flops += 2.0 * t.m * t.n * (double)t.k;
        ln.gemm_bytes += 8.0 * ((double)t.m * t.k + (double)t.k * t.n + (1.0 + (t.beta != 0.0)) * t.m * t.n);
      }
      ln.nrow = (int)rows.size();
      ln.ncol = (int)cols.size();
      rows.insert(rows.end(), cols.begin(), cols.end());
      ln.table_off = push(thin.data(), thin.size() * sizeof(GemmTask));
      ln.ids_off = push(rows.data(), rows.size() * sizeof(int));
      launches.push_back(ln);
    }
  };
  auto outView = [&](int l, long long z) -> View { return out_view(l, z); };

  // ---- formation, levels 1..L ----
  for (int l = 1; l <= L; ++l) {
    const Dims& d = dims[l];
    if (collapse && l == L) break;  // emitted with level L-1
    if (collapse && l == L - 1) {
      emit_two_level_formation(lazy_kernels);
      break;
    }
    for (int side = 0; side < 2; ++side) {
      const auto& form = side == 0 ? formU : formV;
      if (form.empty()) continue;
      const int nin = side == 0 ? M * K : K * Nb;
      const int nout = (int)form.size();
      const long long rows = side == 0 ? d.P : d.Q, cols = side == 0 ? d.Q : d.N;
      if (rows <= 0 || cols <= 0) continue;
      std::vector<char> tab;
      std::vector<int> node_ids;
      const size_t nb = lincomb_node_bytes(nin, nout);
      bool aligned = (cols % 2) == 0;
      int count = 0;
      double writes = 0;
      std::vector<double> mat_count(nout, 0.0);  // nodes materialising output o
      for (long long zp = 0; zp < nodes_at[l - 1]; ++zp) {
        if (!needed[l - 1][zp]) continue;
        bool any = false;
        for (int o = 0; o < nout; ++o) any |= needed[l][zp * R + form[o]] != 0;
        if (!any) continue;
        const View par = side == 0 ? opA(l - 1, zp, rootA) : opB(l - 1, zp, rootB);
        std::vector<char> e(nb, 0);
        auto** in = reinterpret_cast<const double**>(e.data());
        auto** out = reinterpret_cast<double**>(e.data() + sizeof(void*) * nin);
        auto* lds = reinterpret_cast<long long*>(e.data() + sizeof(void*) * (nin + nout));
        for (int i = 0; i < nin; ++i) {
          const long long off = side == 0 ? (i / K) * d.P * par.ld + (i % K) * d.Q : (i / Nb) * d.Q * par.ld + (i % Nb) * d.N;
          in[i] = par.ptr + off;
          aligned &= al16(in[i]);
        }
        for (int o = 0; o < nout; ++o) {
          const long long z = zp * R + form[o];
          const long long offv = side == 0 ? offS[l][z] : offT[l][z];
          out[o] = needed[l][z] && offv >= 0 ? ws + offv : nullptr;
          if (out[o]) writes += 1, mat_count[o] += 1;
        }
        lds[0] = par.ld;
        lds[1] = side == 0 ? ldS[l] : ldT[l];
        aligned &= (lds[0] % 2 == 0) && (lds[1] % 2 == 0);
        tab.insert(tab.end(), e.begin(), e.end());
        node_ids.push_back((int)zp);
        ++count;
      }
      if (!count) continue;
      if (emit_mcse(side == 0 ? Launch::FORM_A : Launch::FORM_B, l, side, tab, nin, nout, count, rows, cols, aligned,
                    node_ids))
        continue;
      Launch ln;
      ln.node_ids = node_ids;
      ln.kind = side == 0 ? Launch::FORM_A : Launch::FORM_B;
      ln.level = l;
      ln.count = count;
      ln.rows = rows;
      ln.cols = cols;
      ln.aligned16 = aligned;
      if (!lazy_kernels) ln.kern = kernel(side, aligned ? 2 : 1);
      const auto k = kernel(side, 2);  // cost model is vec-independent
      const LincombCost c = lincomb_cost(*k);
      const double elems = (double)rows * cols;
      ln.elem_adds = c.adds_per_elem * elems * count;
      if (opt.strategy == FMM_ADD_PAIRWISE) {
        // per materialised chain of n terms: a copy (1 read, 1 write), then n - 1 daxpy passes
        // (2 reads, 1 write each) -- P:638-640
        ln.elem_reads = ln.elem_writes = 0;
        for (int o = 0; o < nout; ++o) {
          const double n = lincomb_out_terms(*k, o);
          ln.elem_reads += mat_count[o] * (2 * n - 1) * elems;
          ln.elem_writes += mat_count[o] * n * elems;
        }
      } else {
        // streaming: every used input once; write-once: the sum of chain lengths per node
        ln.elem_reads = c.reads_per_elem * elems * count;
        ln.elem_writes = writes * elems;
      }
      ln.table_off = push(tab.data(), tab.size());
      launches.push_back(ln);
    }
  }

  // ---- leaf GEMMs ----
  {
    std::vector<GemmTask> tasks;
    const Dims& d = dims[L];
    for (long long z = 0; z < nodes_at[L]; ++z) {
      const long long r0 = leaf_r0[z], r1 = leaf_r1[z];
      if (r1 <= r0) continue;
      const View a = opA(L, z, rootA), b = opB(L, z, rootB), c = outView(L, z);
      GemmTask t{};
      t.A = a.ptr + r0 * a.ld;
      t.B = b.ptr;
      t.C = c.ptr + r0 * c.ld;
      t.lda = a.ld;
      t.ldb = b.ld;
      t.ldc = c.ld;
      t.m = (int)(r1 - r0);
      t.n = (int)d.N;
      t.k = (int)d.Q;
      t.alpha = a.sigma * b.sigma;
      t.beta = 0.0;
      t.node = (int)(z / R);
      t.aux = (int)(z % R);
      if (t.m > 0 && t.n > 0) tasks.push_back(t);
    }
    if (L == 0 && opt.shard_count > 1) {
      // the root is the only leaf: a shard writes its rows of C and zeros in the rest (k = 0 tasks;
      // deeper levels get zeros from the zero-initialised workspace instead)
      const View c = outView(0, 0);
      auto zero = [&](long long r0, long long r1) {
        if (r1 <= r0 || d.N <= 0) return;
        GemmTask t{};
        t.A = rootA.ptr;
        t.B = rootB.ptr;
        t.C = c.ptr + r0 * c.ld;
        t.lda = rootA.ld;
        t.ldb = rootB.ld;
        t.ldc = c.ld;
        t.m = (int)(r1 - r0);
        t.n = (int)d.N;
        t.k = 0;
        t.alpha = 1.0;
        t.beta = 0.0;
        t.node = -1;
        tasks.push_back(t);
      };
      const long long r0 = leaf_r0[0], r1 = leaf_r1[0];
      if (r1 <= r0) zero(0, d.P);
      else zero(0, r0), zero(r1, d.P);
    }
    if (k3f) emit_k3f(tasks, lazy_kernels);
    else emit_gemm(Launch::GEMM, L, tasks);
  }

  // ---- assembly and peel strips, levels L..1 ----
  for (int l = L; l >= 1; --l) {
    const Dims& d = dims[l];
    const Dims& dp = dims[l - 1];
    if (collapse_asm && l == L) emit_two_level_assembly(lazy_kernels);
    if (!(collapse_asm && l >= L - 1) && !(k3f && l == L) && d.P > 0 && d.N > 0) {
      std::vector<char> tab;
      std::vector<int> node_ids;
      const int nin = R, nout = M * Nb;
      const size_t nb = lincomb_node_bytes(nin, nout);
      bool aligned = (d.N % 2) == 0;
      int count = 0;
      for (long long zp = 0; zp < nodes_at[l - 1]; ++zp) {
        if (!needed[l - 1][zp]) continue;
        const View par = outView(l - 1, zp);
        std::vector<char> e(nb, 0);
        auto** in = reinterpret_cast<const double**>(e.data());
        auto** out = reinterpret_cast<double**>(e.data() + sizeof(void*) * nin);
        auto* lds = reinterpret_cast<long long*>(e.data() + sizeof(void*) * (nin + nout));
        for (int r = 0; r < R; ++r) {
          in[r] = skip_absent() && !needed[l][zp * R + r] ? nullptr : outView(l, zp * R + r).ptr;
          aligned &= al16(in[r]);
        }
        for (int k = 0; k < nout; ++k) {
          out[k] = par.ptr + (k / Nb) * d.P * par.ld + (k % Nb) * d.N;
          aligned &= al16(out[k]);
        }
        lds[0] = ldM[l];
        lds[1] = par.ld;
        aligned &= (lds[0] % 2 == 0) && (lds[1] % 2 == 0);
        tab.insert(tab.end(), e.begin(), e.end());
        node_ids.push_back((int)zp);
        ++count;
      }
      if (count && !emit_mcse(Launch::ASSEMBLE, l, 2, tab, nin, nout, count, d.P, d.N, aligned, node_ids)) {
        Launch ln;
        ln.node_ids = node_ids;
        ln.kind = Launch::ASSEMBLE;
        ln.level = l;
        ln.nin = nin;
        ln.nout = nout;
        ln.count = count;
        ln.rows = d.P;
        ln.cols = d.N;
        ln.aligned16 = aligned;
        if (!lazy_kernels) ln.kern = kernel(2, aligned ? 2 : 1);
        const LincombCost c = lincomb_cost(*kernel(2, 2));
        const double elems = (double)d.P * d.N;
        ln.elem_adds = c.adds_per_elem * elems * count;
        ln.elem_reads = c.reads_per_elem * elems * count;
        ln.elem_writes = c.writes_per_elem * elems * count;
        ln.table_off = push(tab.data(), tab.size());
        launches.push_back(ln);
      }
    }
    // peel strips of the level-(l-1) nodes: (a) C'[0:P',0:N'] += A[:,Q':Q] B[Q':Q,0:N'],
    // (b) C[P':P,:] = A[P':P,:] B, (c) C[0:P',N':N] = A[0:P',:] B[:,N':N]
    std::vector<GemmTask> tasks;
    for (long long zp = 0; zp < nodes_at[l - 1]; ++zp) {
      if (l - 1 == 0 && !strip_owner[0][0] && opt.shard_count > 1) {
        // a shard that does not own the root's strips still writes its partial C there: zeros
        // (k = 0 tasks); deeper strip regions live in the zero-initialised workspace
        const View c = outView(0, 0);
        auto zero = [&](double* pc, long long m, long long n) {
          if (m <= 0 || n <= 0) return;
          GemmTask t{};
          t.A = rootA.ptr;
          t.B = rootB.ptr;
          t.C = pc;
          t.lda = rootA.ld;
          t.ldb = rootB.ld;
          t.ldc = c.ld;
          t.m = (int)m;
          t.n = (int)n;
          t.k = 0;
          t.alpha = 1.0;
          t.beta = 0.0;
          tasks.push_back(t);
        };
        if (dp.P1 < dp.P) zero(c.ptr + dp.P1 * c.ld, dp.P - dp.P1, dp.N);
        if (dp.N1 < dp.N) zero(c.ptr + dp.N1, dp.P1, dp.N - dp.N1);
        continue;
      }
      if (!strip_owner[l - 1][zp]) continue;
      const View a = opA(l - 1, zp, rootA), b = opB(l - 1, zp, rootB), c = outView(l - 1, zp);
      const double alpha = a.sigma * b.sigma;
      auto add = [&](const double* pa, const double* pb, double* pc, long long m, long long n, long long k, double beta) {
        if (m <= 0 || n <= 0) return;
        GemmTask t{};
        t.A = pa;
        t.B = pb;
        t.C = pc;
        t.lda = a.ld;
        t.ldb = b.ld;
        t.ldc = c.ld;
        t.m = (int)m;
        t.n = (int)n;
        t.k = (int)k;
        t.alpha = alpha;
        t.beta = beta;
        tasks.push_back(t);
      };
      if (dp.Q1 < dp.Q) add(a.ptr + dp.Q1, b.ptr + dp.Q1 * b.ld, c.ptr, dp.P1, dp.N1, dp.Q - dp.Q1, 1.0);
      if (dp.P1 < dp.P) add(a.ptr + dp.P1 * a.ld, b.ptr, c.ptr + dp.P1 * c.ld, dp.P - dp.P1, dp.N, dp.Q, 0.0);
      if (dp.N1 < dp.N) add(a.ptr, b.ptr + dp.N1, c.ptr + dp.N1, dp.P1, dp.N - dp.N1, dp.Q, 0.0);
    }
    emit_gemm(Launch::STRIPS, l - 1, tasks);
  }
  fuse_leaf_level(lazy_kernels);
  chunk_final_assembly();
}

void fmm_plan_s::chunk_final_assembly() {
  dist_chunked = false;
  if (!dist_comm || opt.dist_chunks <= 1 || L < 1) return;
  int ia = -1, nasm = 0;
  for (int q = 0; q < (int)launches.size(); ++q)
    if (launches[q].kind == Launch::ASSEMBLE && launches[q].level == 1) ia = q, ++nasm;
  // one streaming assembly writes C (memory-CSE strategies emit several launches), over the root only
  if (ia < 0 || nasm != 1 || launches[ia].count != 1 || launches[ia].nin <= 0) return;
  const Dims& d0 = dims[0];
  if (d0.Q1 < d0.Q) return;  // strip (a) would add into C's core after the assembly
  for (int q = ia + 1; q < (int)launches.size(); ++q)  // only level-0 strips follow it
    if (!((launches[q].kind == Launch::STRIPS || launches[q].kind == Launch::SKINNY) && launches[q].level == 0)) return;
  const Launch base = launches[ia];
  const long long rows = base.rows;
  const int nch = (int)std::min<long long>(opt.dist_chunks, std::max<long long>(rows, 1));
  const size_t nb = lincomb_node_bytes(base.nin, base.nout);
  std::vector<char> entry(h_tab.begin() + base.table_off, h_tab.begin() + base.table_off + nb);
  auto** in0 = reinterpret_cast<const double**>(entry.data());
  auto** out0 = reinterpret_cast<double**>(entry.data() + sizeof(void*) * base.nin);
  const auto* lds0 = reinterpret_cast<const long long*>(entry.data() + sizeof(void*) * (base.nin + base.nout));
  // first row of C (plan orientation) of every output block
  std::vector<long long> starts;
  for (int k = 0; k < base.nout; ++k) starts.push_back((long long)(out0[k] - cur_C) / std::max<long long>(cur_ldc, 1));
  std::sort(starts.begin(), starts.end());
  starts.erase(std::unique(starts.begin(), starts.end()), starts.end());
  std::vector<Launch> chunks;
  std::vector<std::pair<long long, long long>> covered;
  for (int j = 0; j < nch; ++j) {
    const long long r0 = rows * j / nch, r1 = rows * (j + 1) / nch;
    if (r1 <= r0) continue;
    std::vector<char> e = entry;
    auto** in = reinterpret_cast<const double**>(e.data());
    auto** out = reinterpret_cast<double**>(e.data() + sizeof(void*) * base.nin);
    for (int i = 0; i < base.nin; ++i)
      if (in0[i]) in[i] = in0[i] + r0 * lds0[0];
    for (int k = 0; k < base.nout; ++k) out[k] = out0[k] + r0 * lds0[1];
    Launch ln = base;
    ln.rows = r1 - r0;
    ln.table_off = push_tab(e.data(), e.size());
    const double f = (double)(r1 - r0) / (double)rows;
    ln.elem_adds = base.elem_adds * f, ln.elem_reads = base.elem_reads * f, ln.elem_writes = base.elem_writes * f;
    ln.reduce_rows.clear();
    for (long long s0 : starts) {
      if (!ln.reduce_rows.empty() && ln.reduce_rows.back().second == s0 + r0) ln.reduce_rows.back().second = s0 + r1;
      else ln.reduce_rows.push_back({s0 + r0, s0 + r1});
      covered.push_back({s0 + r0, s0 + r1});
    }
    chunks.push_back(ln);
  }
  // rows no chunk covers (the bottom peel strip (b)) are reduced once everything is written
  std::sort(covered.begin(), covered.end());
  Launch tail;
  tail.kind = Launch::REDUCE;
  tail.level = 0;
  long long at = 0;
  for (const auto& c : covered) {
    if (c.first > at) tail.reduce_rows.push_back({at, c.first});
    at = std::max(at, c.second);
  }
  if (at < d0.P) tail.reduce_rows.push_back({at, d0.P});
  // level-0 strips (b) and (c) write C outside the assembled core: launch them first
  std::vector<Launch> out(launches.begin(), launches.begin() + ia);
  out.insert(out.end(), launches.begin() + ia + 1, launches.end());
  out.insert(out.end(), chunks.begin(), chunks.end());
  if (!tail.reduce_rows.empty()) out.push_back(tail);
  launches.swap(out);
  dist_chunked = true;
}

// K3f (SURVEY 8(a) a6 option 4 with a fixed-function reduction): the level-L assembly
// C_k = sum_r w_kr M_r of every level-(L-1) node moves into the leaf GEMM's epilogue.  Each leaf tile
// is reduce-added (TMA, fp64 add in L2) into the sub-blocks k of its parent's output with w_kr != 0:
// +acc where w = 1, -acc where w = -1.  The parents' outputs are zeroed first.
void fmm_plan_s::emit_k3f(std::vector<GemmTask>& tasks, bool lazy_kernels) {
  const Dims& dp = dims[L - 1];
  const Dims& d = dims[L];
  const int Nb = alg->N;
  auto push = [&](const void* ptr, size_t n) { return push_tab(ptr, n); };
  // zero the outputs of the needed level-(L-1) nodes (their core and strips; strips rewrite theirs)
  Launch zl;
  zl.kind = Launch::ZERO;
  zl.level = L - 1;
  for (long long zp = 0; zp < nodes_at[L - 1]; ++zp) {
    if (!needed[L - 1][zp]) continue;
    const View o = out_view(L - 1, zp);
    zl.zero_blocks.push_back({(long long)reinterpret_cast<uintptr_t>(o.ptr), o.ld, dp.P, dp.N});
    zl.elem_writes += (double)dp.P * dp.N;
  }
  zl.count = (int)zl.zero_blocks.size();
  launches.push_back(zl);
  if (tasks.empty()) return;
  if (!lazy_kernels) {
    bool ok = gemm_tma_eligible(tasks);
    for (long long zp = 0; zp < nodes_at[L - 1]; ++zp) {
      if (!needed[L - 1][zp]) continue;
      const View o = out_view(L - 1, zp);
      ok &= al16(o.ptr) && o.ld % 2 == 0;
    }
    if (!ok)
      throw Error(FMM_E_UNSUPPORTED, "fuse_output (K3f) needs 16-byte aligned A, B, C with even leading dimensions (TMA)");
  }
  Launch ln;
  ln.kind = Launch::GEMM;
  ln.level = L;
  ln.k3f = true;
  ln.tma = !lazy_kernels;
  ln.bn = K3F_BN;
  ln.tiles = gemm_prepare(tasks, 128, ln.bn);
  gemm_uniform_grid(tasks, &ln.uni_tm, &ln.uni_tn);
  ln.count = (int)tasks.size();
  ln.aligned16 = gemm_tasks_aligned16(tasks);
  for (auto& t : tasks) {
    ln.flops += 2.0 * t.m * t.n * (double)t.k;
    ln.gemm_bytes += 8.0 * ((double)t.m * t.k + (double)t.k * t.n);
  }
  ln.table_off = push(tasks.data(), tasks.size() * sizeof(GemmTask));
  {  // operand maps (A, B per task), as every TMA GEMM launch
    std::vector<char> maps(2 * gemm_tma_map_bytes() * tasks.size());
    if (!lazy_kernels) gemm_tma_maps(tasks, maps.data(), BK_K3F);
    ln.maps_off = push(lazy_kernels ? nullptr : maps.data(), maps.size());
  }
  {  // one target map per parent node: its output block, dims[L-1].P x dims[L-1].N
    const size_t mb = gemm_tma_map_bytes();
    std::vector<char> tm(mb * (size_t)nodes_at[L - 1], 0);
    if (!lazy_kernels)
      for (long long zp = 0; zp < nodes_at[L - 1]; ++zp) {
        if (!needed[L - 1][zp]) continue;
        const View o = out_view(L - 1, zp);
        gemm_k3f_target_map(tm.data() + mb * zp, o.ptr, dp.P, dp.N, o.ld);
      }
    ln.k3f_maps_off = push(lazy_kernels ? nullptr : tm.data(), tm.size());
  }
  {  // per leaf column r of W: its targets (row / column offset of sub-block k in the parent, sign)
    std::vector<int> count(R, 0);
    std::vector<K3fTarget> tg((size_t)R * K3F_MAX_TARGETS);
    for (int r = 0; r < R; ++r)
      for (int k = 0; k < alg->M * Nb; ++k) {
        const double w = alg->Wd[(size_t)k * R + r];
        if (w == 0.0) continue;
        K3fTarget& x = tg[(size_t)r * K3F_MAX_TARGETS + count[r]++];
        x.row_off = (int)((k / Nb) * d.P);
        x.col_off = (int)((k % Nb) * d.N);
        x.sign = w > 0 ? 1 : -1;
        x.pad = 0;
      }
    if (const char* e = getenv("FMM_K3F_MAX_TARGETS"))  // timing diagnostics only: drops targets (wrong C)
      for (int& cnt : count) cnt = std::min(cnt, atoi(e));
    ln.k3f_count_off = push(count.data(), count.size() * sizeof(int));
    ln.k3f_targets_off = push(tg.data(), tg.size() * sizeof(K3fTarget));
    // the reduce-adds, as output traffic: every leaf element once per target
    for (const auto& t : tasks) ln.elem_writes += (double)t.m * t.n * count[t.aux];
  }
  launches.push_back(ln);
}

// The fused leaf level (fmm_gemm_tma.cu, FUSED kernel).  Jobs: formation (F) of the level-L S / T
// of one parent node (level L-1) over a row range, assembly (A) of the parent's C / M sub-blocks
// from its R leaf products over a row range.  Phase 0 = F jobs of the first parent (every warp of
// the GPU helps: no leaf product can start before them); phase 1 = F of the other parents and
// the A jobs, interleaved so formation stays LOOKAHEAD parents ahead of the GEMM and assembly
// follows the GEMM's parent-major tile order.  Chains are the coefficient rows without CSE,
// ascending input index (the oracle's order, R8).
void fmm_plan_s::fuse_leaf_level(bool lazy_kernels) {
  if (!fuse || L < 1 || opt.strategy != FMM_ADD_STREAMING) return;
  int ia = -1, ib = -1, ig = -1, ias = -1;
  for (int q = 0; q < (int)launches.size(); ++q) {
    const Launch& ln = launches[q];
    if (ln.level != L) continue;
    if (ln.kind == Launch::FORM_A) ia = q;
    else if (ln.kind == Launch::FORM_B) ib = q;
    else if (ln.kind == Launch::GEMM) ig = q;
    else if (ln.kind == Launch::SKINNY) return;  // thin leaves: no fusion
    else if (ln.kind == Launch::ASSEMBLE) ias = q;
  }
  if (ig < 0 || ias < 0) return;
  if (!lazy_kernels && !launches[ig].tma) return;
  if (fuse_bg) {  // the producer warps' input staging (256 bytes per input, fused_bg_stage_bytes) must fit
    const int nin = std::max(std::max(alg->M * alg->K, alg->K * alg->N), R);
    if (gemm_fused_smem_bytes(launches[ig].bn, launches[ig].bk, 256 * nin) > gemm_max_smem_bytes()) return;
  }
  const long long np = nodes_at[L - 1];
  Launch fz = launches[ig];
  fz.kind = Launch::FUSED;
  fz.np = (int)np;
  // programs: the absorbed launches' node tables and chains (the same generated chains as their
  // separate K1/K3 kernels)
  std::vector<int> prog_src;
  std::vector<int> sides;
  if (ia >= 0) prog_src.push_back(ia), sides.push_back(0);
  if (ib >= 0) prog_src.push_back(ib), sides.push_back(1);
  prog_src.push_back(ias), sides.push_back(2);
  fz.nprogs = (int)prog_src.size();
  for (int q = 0; q < fz.nprogs; ++q) {
    const Launch& ln = launches[prog_src[q]];
    const int nin = sides[q] == 0 ? alg->M * alg->K : sides[q] == 1 ? alg->K * alg->N : R;
    const int nout = sides[q] == 0 ? (int)formU.size() : sides[q] == 1 ? (int)formV.size() : alg->M * alg->N;
    fz.prog_node_off[q] = ln.table_off;
    fz.prog_node_bytes[q] = (int)lincomb_node_bytes(nin, nout);
    fz.prog_cols[q] = (int)ln.cols;
    fz.prog_vec2[q] = ln.aligned16 ? 1 : 0;
    fz.elem_adds += ln.elem_adds;
    fz.elem_reads += ln.elem_reads;
    fz.elem_writes += ln.elem_writes;
  }
  const int pA = fz.nprogs - 1;
  // jobs per parent; phase 0 = formation of the parent of the first leaf product in tile order
  const GemmTask* tk = reinterpret_cast<const GemmTask*>(h_tab.data() + fz.table_off);
  const int first_node = fz.count > 0 ? tk[0].node : -1;
  std::vector<int> ready_target(np, 0), tiles_target(np, 0);
  for (int q = 0; q < fz.count; ++q)
    if (tk[q].node >= 0 && tk[q].node < np) tiles_target[tk[q].node] += tk[q].tiles_m * tk[q].tiles_n;
  std::vector<std::vector<FusedJob>> fjobs0(np), fjobs(np), ajobs(np);
  for (int pi = 0; pi < fz.nprogs; ++pi) {
    const Launch& ln = launches[prog_src[pi]];
    const bool is_a = pi == pA;
    for (int e = 0; e < (int)ln.node_ids.size(); ++e) {
      const int zp = ln.node_ids[e];
      const bool first = !is_a && zp == first_node;
      // a job is a few rows of one warp (about 1-4 K element positions): enough jobs per parent to
      // spread over every addition warp, none long against the parent's share of the GEMM
      const int per = std::max(1, (first ? 512 : 2048) / std::max(1, (int)ln.cols));
      for (int r0 = 0; r0 < (int)ln.rows; r0 += per) {
        FusedJob j{pi, e, r0, std::min(per, (int)ln.rows - r0), zp, is_a ? 1 : 0};
        if (is_a) ajobs[zp].push_back(j);
        else {
          (first ? fjobs0 : fjobs)[zp].push_back(j);
          ++ready_target[zp];
        }
      }
    }
  }
  std::vector<FusedJob> jobs;
  for (long long zp = 0; zp < np; ++zp) jobs.insert(jobs.end(), fjobs0[zp].begin(), fjobs0[zp].end());
  fz.njobs0 = (int)jobs.size();
  const long long LOOKAHEAD = 2;
  for (long long zp = 0; zp < np; ++zp) {
    jobs.insert(jobs.end(), fjobs[zp].begin(), fjobs[zp].end());
    if (zp >= LOOKAHEAD) jobs.insert(jobs.end(), ajobs[zp - LOOKAHEAD].begin(), ajobs[zp - LOOKAHEAD].end());
  }
  for (long long zp = std::max(0LL, np - LOOKAHEAD); zp < np; ++zp) jobs.insert(jobs.end(), ajobs[zp].begin(), ajobs[zp].end());
  fz.njobs = (int)jobs.size();
  // spatial split of the SMs: k addition CTAs on their own SMs (the FP64 ALU and the DMMA path
  // are one pipe), the rest run leaf tiles; k balances the leaf flops at the per-SM DMMA rate
  // against the absorbed addition bytes at the per-SM rate of an addition CTA
  {
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
    cudaGetLastError();
    const double bytes = 8.0 * (fz.elem_reads + fz.elem_writes), fl = fz.flops;
    // measured (round 1): ~245 GFLOP/s per GEMM SM, ~80 GB/s per addition SM (loads + stores)
    const double F_SM = 245e9, B_SM = 80e9;
    int best_k = 1;
    double best_t = 1e300;
    for (int k = 1; k <= sms / 3; ++k) {
      const double t = std::max(fl / ((sms - k) * F_SM), bytes / (k * B_SM));
      if (t < best_t) best_t = t, best_k = k;
    }
    if (const char* e = getenv("FMM_FUSE_ADD_CTAS")) best_k = std::max(1, std::min(sms - 1, atoi(e)));
    fz.gemm_ctas = fuse_bg ? sms : sms - best_k;  // background mode: every SM runs leaf tiles
  }
  auto push = [&](const void* p, size_t n) {
    size_t off = h_tab.size();
    h_tab.resize(align256(off + n));
    if (n) std::memcpy(h_tab.data() + off, p, n);
    return off;
  };
  fz.jobs_off = push(jobs.data(), jobs.size() * sizeof(FusedJob));
  std::vector<int> targets(ready_target);
  targets.insert(targets.end(), tiles_target.begin(), tiles_target.end());
  fz.targets_off = push(targets.data(), targets.size() * sizeof(int));
  if (!lazy_kernels) {
    std::vector<LincombSpec> specs;
    for (int q = 0; q < fz.nprogs; ++q) specs.push_back(lincomb_spec(*kernel(sides[q], 2)));
    fz.fk = fused_get(specs, fz.bn, fz.bk, fuse_bg);
  }
  // replace: GEMM -> FUSED; drop the absorbed formation / assembly launches
  launches[ig] = fz;
  std::vector<Launch> keep;
  for (int q = 0; q < (int)launches.size(); ++q)
    if (q != ia && q != ib && q != ias) keep.push_back(launches[q]);
  launches.swap(keep);
}

// Write-once / pairwise with CSE: the greedy length-two subexpressions Y_t = x_a + r x_b
// (the same ones the streaming kernels keep in registers) are written to memory once per node by
// their own launches, in creation order (a later Y may use an earlier one), then the main launch
// evaluates every chain over the inputs and the Y_t.  Each Y_t has the node's input leading
// dimension, so one ld serves all inputs of the main launch.  Returns false (nothing emitted)
// for streaming, without CSE, or when the chains share no subexpression.
bool fmm_plan_s::emit_mcse(Launch::Kind kind, int level, int side, const std::vector<char>& tab, int nin, int nout,
                           int count, long long rows, long long cols, bool aligned, const std::vector<int>& node_ids) {
  if (opt.strategy == FMM_ADD_STREAMING || !opt.cse) return false;
  std::vector<std::tuple<int, int, double>> temps;
  std::vector<std::vector<std::pair<int, double>>> outs;
  const LincombSpec base = spec_for(side, 2);
  lincomb_cse_program(base, &temps, &outs);
  const int T = (int)temps.size();
  if (T == 0) return false;
  const size_t nb = lincomb_node_bytes(nin, nout);
  const int vec = aligned ? 2 : 1;
  const double elems = (double)rows * cols;
  // per node: its input pointers, output pointers, leading dimensions; temporaries from the arena
  std::vector<std::vector<const double*>> var(count);  // nin inputs then T temporaries
  std::vector<std::vector<double*>> outp(count);
  std::vector<long long> ldi(count), ldo(count);
  for (int z = 0; z < count; ++z) {
    const char* e = tab.data() + (size_t)z * nb;
    const double* const* in = reinterpret_cast<const double* const*>(e);
    double* const* out = reinterpret_cast<double* const*>(e + sizeof(void*) * nin);
    auto* lds = reinterpret_cast<const long long*>(e + sizeof(void*) * (nin + nout));
    ldi[z] = lds[0];
    ldo[z] = lds[1];
    var[z].assign(in, in + nin);
    outp[z].assign(out, out + nout);
    for (int t = 0; t < T; ++t) var[z].push_back(scratch_take(rows * ldi[z]));
  }
  auto emit = [&](const LincombSpec& sp, const std::vector<char>& t2, double reads, double writes) {
    Launch ln;
    ln.node_ids = node_ids;
    ln.kind = kind;
    ln.level = level;
    ln.count = count;
    ln.rows = rows;
    ln.cols = cols;
    ln.aligned16 = aligned;
    ln.kern = lincomb_get(sp);
    ln.elem_adds = lincomb_cost(*ln.kern).adds_per_elem * elems * count;
    ln.elem_reads = reads * elems;
    ln.elem_writes = writes * elems;
    ln.table_off = push_tab(t2.data(), t2.size());
    launches.push_back(ln);
  };
  const bool pw = opt.strategy == FMM_ADD_PAIRWISE;
  // the temporaries, Y_t = x_a + r x_b: a two-term chain (pairwise: a copy and one daxpy)
  for (int t = 0; t < T; ++t) {
    LincombSpec sp;
    sp.nin = 2;
    sp.nout = 1;
    sp.coef = {1.0, std::get<2>(temps[t])};
    sp.strategy = opt.strategy;
    sp.cse = 0;
    sp.vec = vec;
    std::vector<char> t2;
    const size_t nb2 = lincomb_node_bytes(2, 1);
    for (int z = 0; z < count; ++z) {
      std::vector<char> e(nb2, 0);
      auto** in = reinterpret_cast<const double**>(e.data());
      auto** out = reinterpret_cast<double**>(e.data() + sizeof(void*) * 2);
      auto* lds = reinterpret_cast<long long*>(e.data() + sizeof(void*) * 3);
      in[0] = var[z][std::get<0>(temps[t])];
      in[1] = var[z][std::get<1>(temps[t])];
      out[0] = const_cast<double*>(var[z][nin + t]);
      lds[0] = ldi[z];
      lds[1] = ldi[z];
      t2.insert(t2.end(), e.begin(), e.end());
    }
    emit(sp, t2, (pw ? 3.0 : 2.0) * count, (pw ? 2.0 : 1.0) * count);
  }
  // the chains over inputs and temporaries
  LincombSpec sp;
  sp.nin = nin + T;
  sp.nout = nout;
  sp.coef.assign((size_t)sp.nin * nout, 0.0);
  for (int o = 0; o < nout; ++o)
    for (const auto& kv : outs[o]) sp.coef[(size_t)o * sp.nin + kv.first] = kv.second;
  sp.strategy = opt.strategy;
  sp.cse = 0;
  sp.vec = vec;
  const size_t nbm = lincomb_node_bytes(sp.nin, nout);
  std::vector<char> tm;
  double reads = 0, writes = 0;
  for (int z = 0; z < count; ++z) {
    std::vector<char> e(nbm, 0);
    auto** in = reinterpret_cast<const double**>(e.data());
    auto** out = reinterpret_cast<double**>(e.data() + sizeof(void*) * sp.nin);
    auto* lds = reinterpret_cast<long long*>(e.data() + sizeof(void*) * (sp.nin + nout));
    for (int v = 0; v < sp.nin; ++v) in[v] = var[z][v];
    for (int o = 0; o < nout; ++o) {
      out[o] = outp[z][o];
      if (!out[o]) continue;
      const double n = (double)outs[o].size();
      reads += pw ? 2 * n - 1 : n;
      writes += pw ? n : 1;
    }
    lds[0] = ldi[z];
    lds[1] = ldo[z];
    tm.insert(tm.end(), e.begin(), e.end());
  }
  emit(sp, tm, reads, writes);
  return true;
}

void fmm_plan_s::emit_two_level_formation(bool lazy_kernels) {
  const int M = alg->M, K = alg->K, Nb = alg->N;
  const Dims &d1 = dims[L - 1], &d2 = dims[L];
  const View rootA{const_cast<double*>(cur_A), cur_lda, 1.0}, rootB{const_cast<double*>(cur_B), cur_ldb, 1.0};
  for (int side = 0; side < 2; ++side) {
    const int rows = side == 0 ? M * K : K * Nb, inner = side == 0 ? K : Nb;
    const auto& idx = side == 0 ? idxU : idxV;
    const long long brow = side == 0 ? d2.P : d2.Q, bcol = side == 0 ? d2.Q : d2.N;
    if (brow <= 0 || bcol <= 0) continue;
    std::vector<char> mat((size_t)R * R, 0);
    bool any_mat = false;
    for (int r1 = 0; r1 < R; ++r1)
      for (int r2 = 0; r2 < R; ++r2) any_mat |= (mat[(size_t)r1 * R + r2] = (idx[r1] >= 0 || idx[r2] >= 0));
    if (!any_mat) continue;
    const int nin = rows * rows, nout = R * R;
    const size_t nb = lincomb_node_bytes(nin, nout);
    std::vector<char> tab;
    std::vector<int> node_ids;
    bool aligned = (bcol % 2) == 0;
    int count = 0;
    double writes = 0;
    for (long long zg = 0; zg < nodes_at[L - 2]; ++zg) {
      if (!needed[L - 2][zg]) continue;
      const View g = side == 0 ? opA(L - 2, zg, rootA) : opB(L - 2, zg, rootB);
      std::vector<char> e(nb, 0);
      auto** in = reinterpret_cast<const double**>(e.data());
      auto** out = reinterpret_cast<double**>(e.data() + sizeof(void*) * nin);
      auto* lds = reinterpret_cast<long long*>(e.data() + sizeof(void*) * (nin + nout));
      bool anyout = false;
      for (int i1 = 0; i1 < rows; ++i1)
        for (int i2 = 0; i2 < rows; ++i2) {
          const long long off = side == 0 ? (i1 / inner) * d1.P * g.ld + (i1 % inner) * d1.Q + (i2 / inner) * d2.P * g.ld + (i2 % inner) * d2.Q
                                          : (i1 / inner) * d1.Q * g.ld + (i1 % inner) * d1.N + (i2 / inner) * d2.Q * g.ld + (i2 % inner) * d2.N;
          in[i1 * rows + i2] = g.ptr + off;
          aligned &= ((reinterpret_cast<uintptr_t>(in[i1 * rows + i2]) & 15) == 0);
        }
      for (int q = 0; q < nout; ++q) {
        const long long z = (zg * R + q / R) * R + q % R;
        const long long offv = side == 0 ? offS[L][z] : offT[L][z];
        out[q] = mat[(size_t)q] && needed[L][z] && offv >= 0 ? ws + offv : nullptr;
        if (out[q]) writes += 1, anyout = true;
      }
      if (!anyout) continue;
      lds[0] = g.ld;
      lds[1] = side == 0 ? ldS[L] : ldT[L];
      aligned &= (lds[0] % 2 == 0) && (lds[1] % 2 == 0);
      tab.insert(tab.end(), e.begin(), e.end());
      node_ids.push_back((int)zg);
      ++count;
    }
    if (!count) continue;
    TwoLevelSpec sp;
    sp.side = side;
    sp.rows = rows;
    sp.R = R;
    sp.X = side == 0 ? alg->Ud : alg->Vd;
    sp.materialize = mat;
    sp.vec = aligned && rows <= 4 ? 2 : 1;  // (MK)^2 > 16 inputs: one element per thread (registers)
    Launch ln;
    ln.kind = side == 0 ? Launch::FORM_A : Launch::FORM_B;
    ln.level = L - 1;
    ln.count = count;
    ln.rows = brow;
    ln.cols = bcol;
    ln.aligned16 = aligned;
    ln.node_ids = node_ids;
    ln.kern = twolevel_get(sp);  // cheap when cached; needed for the cost numbers in dry builds too
    const LincombCost c = lincomb_cost(*ln.kern);
    const double elems = (double)brow * bcol;
    ln.elem_adds = c.adds_per_elem * elems * count;
    ln.elem_reads = c.reads_per_elem * elems * count;
    ln.elem_writes = writes * elems;
    ln.table_off = push_tab(tab.data(), tab.size());
    launches.push_back(ln);
  }
  (void)lazy_kernels;
}

void fmm_plan_s::emit_two_level_assembly(bool lazy_kernels) {
  const int M = alg->M, Nb = alg->N;
  const Dims &d1 = dims[L - 1], &d2 = dims[L];
  if (d2.P <= 0 || d2.N <= 0) return;
  const int rows = M * Nb, nin = R * R, nout = rows * rows;
  const size_t nb = lincomb_node_bytes(nin, nout);
  std::vector<char> tab;
  std::vector<int> node_ids;
  bool aligned = (d2.N % 2) == 0;
  int count = 0;
  for (long long zg = 0; zg < nodes_at[L - 2]; ++zg) {
    if (!needed[L - 2][zg]) continue;
    const View par = out_view(L - 2, zg);
    std::vector<char> e(nb, 0);
    auto** in = reinterpret_cast<const double**>(e.data());
    auto** out = reinterpret_cast<double**>(e.data() + sizeof(void*) * nin);
    auto* lds = reinterpret_cast<long long*>(e.data() + sizeof(void*) * (nin + nout));
    for (int q = 0; q < nin; ++q) {
      in[q] = skip_absent() && !needed[L][zg * R * R + q] ? nullptr : out_view(L, zg * R * R + q).ptr;
      aligned &= ((reinterpret_cast<uintptr_t>(in[q]) & 15) == 0);
    }
    for (int k1 = 0; k1 < rows; ++k1)
      for (int k2 = 0; k2 < rows; ++k2) {
        out[k1 * rows + k2] = par.ptr + (k1 / Nb) * d1.P * par.ld + (k1 % Nb) * d1.N + (k2 / Nb) * d2.P * par.ld + (k2 % Nb) * d2.N;
        aligned &= ((reinterpret_cast<uintptr_t>(out[k1 * rows + k2]) & 15) == 0);
      }
    lds[0] = ldM[L];
    lds[1] = par.ld;
    aligned &= (lds[0] % 2 == 0) && (lds[1] % 2 == 0);
    tab.insert(tab.end(), e.begin(), e.end());
    node_ids.push_back((int)zg);
    ++count;
  }
  if (!count) return;
  TwoLevelSpec sp;
  sp.side = 2;
  sp.rows = rows;
  sp.R = R;
  sp.X = alg->Wd;
  sp.vec = aligned ? 2 : 1;
  sp.skip_null = skip_absent();
  Launch ln;
  ln.kind = Launch::ASSEMBLE;
  ln.level = L - 1;
  ln.nin = nin;
  ln.nout = nout;
  ln.count = count;
  ln.rows = d2.P;
  ln.cols = d2.N;
  ln.aligned16 = aligned;
  ln.node_ids = node_ids;
  ln.kern = twolevel_get(sp);
  const LincombCost c = lincomb_cost(*ln.kern);
  const double elems = (double)d2.P * d2.N;
  ln.elem_adds = c.adds_per_elem * elems * count;
  ln.elem_reads = c.reads_per_elem * elems * count;
  ln.elem_writes = c.writes_per_elem * elems * count;
  ln.table_off = push_tab(tab.data(), tab.size());
  launches.push_back(ln);
  (void)lazy_kernels;
}

namespace {

double predict_seconds(const fmm_alg& a, long long P, long long Q, long long N, int levels, int* used_levels);
std::vector<PlanDims> plan_dims(const fmm_alg& a, long long P, long long Q, long long N, int levels, bool peel_align,
                                bool peel_tiles, bool* tiled);

// R7b's peel: widen the peeled strip so the child block widths Q1 / K and N1 / Nb are even
template <class D>
void peel_even(D& d, int K, int Nb) {
  if ((d.Q1 / K) % 2 == 1 && d.Q / (2 * K) >= 1) d.Q1 = 2 * K * (d.Q / (2 * K));
  if ((d.N1 / Nb) % 2 == 1 && d.N / (2 * Nb) >= 1) d.N1 = 2 * Nb * (d.N / (2 * Nb));
}

void plan_init(fmm_plan_t* p, const fmm_alg* alg, long long P, long long Q, long long Nc, int levels,
               const fmm_plan_options* opt, int device) {
  if (!alg) throw Error(FMM_E_INVALID_ARG, "null algorithm");
  if (P < 0 || Q < 0 || Nc < 0) throw Error(FMM_E_SHAPE, "negative dimension");
  if (P > INT32_MAX || Q > INT32_MAX || Nc > INT32_MAX) throw Error(FMM_E_UNSUPPORTED, "dimension above 2^31-1");
  if (levels < -1 || levels > 8) throw Error(FMM_E_UNSUPPORTED, "levels must be in [0, 8], or -1 (automatic)");
  if (levels == -1) {  // the cutoff rule (Sec. 3.4) by the cost model: the fastest L <= 4
    const bool cm = opt && opt->layout == FMM_COL_MAJOR;
    std::unique_ptr<fmm_alg> t;
    const fmm_alg* a = alg;
    if (cm) t.reset(alg_transpose_prop1(*alg)), a = t.get();
    double best = 1e300;
    levels = 0;
    for (int L = 0; L <= 4; ++L) {
      int used = 0;
      const double tt = predict_seconds(*a, cm ? Nc : P, Q, cm ? P : Nc, L, &used);
      if (used < L) break;
      if (tt < best * (1 - 1e-9)) best = tt, levels = L;
    }
  }
  if (opt) p->opt = *opt;
  else fmm_plan_options_default(&p->opt);
  if (p->opt.shard_count < 1) p->opt.shard_count = 1;
  if (p->opt.shard_rank < 0 || p->opt.shard_rank >= p->opt.shard_count) throw Error(FMM_E_INVALID_ARG, "bad shard_rank");
  if (p->opt.shard_mode != 0 && p->opt.shard_mode != 1) throw Error(FMM_E_INVALID_ARG, "bad shard_mode");
  if (p->opt.layout != FMM_ROW_MAJOR && p->opt.layout != FMM_COL_MAJOR) throw Error(FMM_E_INVALID_ARG, "bad layout");
  if (p->opt.strategy != FMM_ADD_STREAMING && p->opt.strategy != FMM_ADD_WRITE_ONCE &&
      p->opt.strategy != FMM_ADD_PAIRWISE)
    throw Error(FMM_E_INVALID_ARG, "bad strategy");
  p->device = device;
  FMM_CUDA(cudaSetDevice(device));
  if (const char* e = getenv("FMM_NO_TMA")) p->use_tma = !(e[0] == '1');
  if (p->opt.fuse_leaf_level < 0 || p->opt.fuse_leaf_level > 2) throw Error(FMM_E_INVALID_ARG, "bad fuse_leaf_level");
  p->fuse = p->opt.fuse_leaf_level != 0;
  p->fuse_bg = p->opt.fuse_leaf_level == 2;
  if (const char* e = getenv("FMM_FUSE_BG")) {  // experiments: force the background mode on (1) or off (0)
    p->fuse_bg = e[0] == '1';
    p->fuse = p->fuse || p->fuse_bg;
  }
  if (const char* e = getenv("FMM_NO_FUSE")) p->fuse = p->fuse && !(e[0] == '1');
  p->userP = P;
  p->userQ = Q;
  p->userN = Nc;
  p->colmajor = p->opt.layout == FMM_COL_MAJOR;
  if (p->colmajor) {
    p->alg_t.reset(alg_transpose_prop1(*alg));
    p->alg = p->alg_t.get();
    p->P = Nc;
    p->Q = Q;
    p->N = P;
  } else {
    p->alg = alg;
    p->P = P;
    p->Q = Q;
    p->N = Nc;
  }
  const fmm_alg* a = p->alg;
  p->R = a->R;
  const int M = a->M, K = a->K, Nb = a->N, R = a->R;
  // effective levels (R10/R18): stop at a level whose problem is smaller than the base case
  // R7b: keep column-block widths even so sub-block views stay 16-byte aligned (TMA): the column
  // offsets of A's blocks are multiples of Q / K, of B's and C's multiples of N / Nb.  R7c: the
  // tile-aware row peel of the last split, where the cost model predicts it faster.
  p->dims = plan_dims(*a, p->P, p->Q, p->N, levels, p->opt.peel_align != 0, p->opt.peel_tiles != 0, &p->tiled_peel);
  const int L = (int)p->dims.size() - 1;
  p->L = L;
  p->nodes_at.assign(L + 1, 1);
  for (int l = 1; l <= L; ++l) {
    if (p->nodes_at[l - 1] > (1LL << 40) / R) throw Error(FMM_E_UNSUPPORTED, "too many recursion nodes");
    p->nodes_at[l] = p->nodes_at[l - 1] * R;
  }
  if (p->nodes_at[L] > 65535 * 16) throw Error(FMM_E_UNSUPPORTED, "too many leaves");
  // formed / singleton columns
  auto cols = [&](const std::vector<double>& X, int rows, std::vector<int>& form, std::vector<int>& idx,
                  std::vector<int>& sing, std::vector<double>& coef) {
    idx.assign(R, -1);
    sing.assign(R, -1);
    coef.assign(R, 0.0);
    for (int r = 0; r < R; ++r) {
      int nz = 0, last = -1;
      for (int i = 0; i < rows; ++i)
        if (X[(size_t)i * R + r] != 0.0) ++nz, last = i;
      if (nz == 1) {
        sing[r] = last;
        coef[r] = X[(size_t)last * R + r];
      } else {
        idx[r] = (int)form.size();
        form.push_back(r);
      }
    }
  };
  cols(a->Ud, M * K, p->formU, p->idxU, p->singU, p->coefU);
  cols(a->Vd, K * Nb, p->formV, p->idxV, p->singV, p->coefV);
  // collapse the last two levels (sec. 6c) where the streaming two-level pass applies: small base
  // case (the pass keeps (MK)^2 inputs in registers), no peeling at level L-1 (its strips would
  // need the level-(L-1) operands the pass never writes)
  {
    const char* e = getenv("FMM_NO_COLLAPSE");
    const Dims& dl = p->dims[L >= 1 ? L - 1 : 0];
    // (a variant reloading the inputs of larger base cases from L1/L2 was measured 2-40 % slower
    // than one level per launch on c4, c5, c5t: the pass is only worth it with every input in registers)
    const bool can = p->opt.collapse_levels && !(e && e[0] == '1') && L >= 2 && p->opt.strategy == FMM_ADD_STREAMING &&
                     dl.P1 == dl.P && dl.Q1 == dl.Q && dl.N1 == dl.N;
    p->collapse = can && M * K <= 4 && K * Nb <= 4 && M * Nb <= 4;
    if (p->collapse && p->fuse_bg && p->fuse) p->collapse = false;  // the background mode hides the level
    if (p->collapse) p->fuse = false;
    p->collapse_asm = p->collapse;
    // the formation alone for base cases with up to 9 x 9 inputs per position (MK, KN <= 9: c4, c5):
    // one thread keeps the (MK)^2 inputs of a position in registers (one element, not two); the
    // (MN)^2 outputs of the assembly do not fit, so it stays one level per launch.  Measured
    // (sec. 6c): c5 -0.4 %, but c4's B side runs at 2.4 TB/s (A side 5.3), so c4 loses 2 %: only on
    // request (FMM_COLLAPSE_FORM=1)
    const char* cf = getenv("FMM_COLLAPSE_FORM");
    if (!p->collapse && can && !p->fuse && M * K <= 9 && K * Nb <= 9 && cf && cf[0] == '1') p->collapse = true;
    // the assembly alone for larger base cases (MN <= 16): the wide warp-per-column kernel (sec. 6g).
    // It halves the assembly's HBM bytes but runs shared-memory bound at about half the HBM rate, so
    // it measured slower than the two separate levels on c4 and c5t: only on request (FMM_WIDE_ASM=1)
    const char* w = getenv("FMM_WIDE_ASM");
    if (!p->collapse_asm && w && w[0] == '1' && p->opt.collapse_levels && !(e && e[0] == '1') && !p->fuse && L >= 2 &&
        p->opt.strategy == FMM_ADD_STREAMING && M * Nb <= 16 && dl.P1 == dl.P && dl.Q1 == dl.Q && dl.N1 == dl.N)
      p->collapse_asm = true;
  }
  // K3f (fuse_output): W entries 0 / +-1 (the staged tile is added as +acc or -acc), MN <= 16
  // targets per leaf, one shard (each leaf whole), the plain TMA leaf GEMM.  It replaces the
  // collapsed levels (whose assembly reads the leaf products) and the fused leaf level.
  {
    const char* e = getenv("FMM_K3F");
    bool want = e ? e[0] == '1' : p->opt.fuse_output != 0;
    bool unit = true;
    for (double w : a->Wd) unit &= (w == 0.0 || w == 1.0 || w == -1.0);
    if (want && L >= 1 && unit && M * Nb <= K3F_MAX_TARGETS && p->opt.shard_count == 1 && p->use_tma) {
      p->k3f = true;
      p->collapse = false;
      p->collapse_asm = false;
      p->fuse = false;
    }
  }
  // small_fused (sec. 6h): one launch for a one-level plan whose leaf products would leave most
  // SMs idle.  The leaf GEMM tiles are 128 x 128 at most; below one per SM the step is launch bound.
  {
    const char* e = getenv("FMM_NO_SMALL");
    // the one launch reads A and B with 8-byte copies, so R7b's alignment peel is not needed: the
    // paper's minimal peeling decides whether the top level divides exactly
    std::vector<Dims> dd = p->dims;
    if (L == 1 && p->opt.peel_align) {
      bool tp = false;
      dd = plan_dims(*a, p->P, p->Q, p->N, levels, false, false, &tp);
    }
    const Dims& d0 = dd[0];
    int max_nu = 0, max_nv = 0;
    for (int r = 0; r < R; ++r) {
      int nu = 0, nv = 0;
      for (int i = 0; i < M * K; ++i) nu += a->Ud[(size_t)i * R + r] != 0.0;
      for (int j = 0; j < K * Nb; ++j) nv += a->Vd[(size_t)j * R + r] != 0.0;
      max_nu = std::max(max_nu, nu), max_nv = std::max(max_nv, nv);
    }
    int kc = 0, g = 0, nw = 0, nuv = 0, nvv = 0;
    for (double w : a->Wd) nw += w != 0.0;
    for (double u : a->Ud) nuv += u != 0.0;
    for (double v : a->Vd) nvv += v != 0.0;
    if (nw <= SMALL_MAX_W && nuv <= SMALL_MAX_UV && nvv <= SMALL_MAX_UV && R <= SMALL_MAX_R && M * Nb <= SMALL_MAX_R &&
        p->opt.small_fused && !(e && e[0] == '1') && L == 1 && (int)dd.size() == 2 && d0.P1 == d0.P && d0.Q1 == d0.Q &&
        d0.N1 == d0.N && p->opt.strategy == FMM_ADD_STREAMING && p->opt.shard_count == 1 && !p->dist_comm && !p->p2p && !p->k3f && !p->fuse && M * K <= 64 &&
        K * Nb <= 64 && M * Nb <= 64 && R <= 128 && small_config(max_nu, max_nv, (int)std::min<long long>(dd[1].Q, 1 << 30), R, &kc, &g)) {
      const Dims& d = dd[1];
      const long long gemm_tiles = (long long)R * ((d.P + 127) / 128) * ((d.N + 127) / 128);
      const int T = small_tile();
      const long long tiles = ((d.P + T - 1) / T) * ((d.N + T - 1) / T);
      if (d.P >= 1 && d.Q >= 1 && d.N >= 1 && d.Q < (1LL << 30) && gemm_tiles < gemm_sm_count() && tiles * R < (1LL << 31)) {
        p->small = true;
        p->dims = dd;
        FMM_CUDA(cudaMalloc(&p->small_M, (size_t)tiles * R * T * T * sizeof(double)));
        FMM_CUDA(cudaMalloc(&p->small_cnt, 2 * (size_t)tiles * sizeof(unsigned)));
        FMM_CUDA(cudaMemset(p->small_cnt, 0, 2 * (size_t)tiles * sizeof(unsigned)));
      }
    }
    // L = 0 below the cutoff: the classical product through the same one launch (base case
    // <1,1,1;1>, each CTA writes its 32 x 32 tile of C) when the GEMM's 128-row tiles would leave
    // most SMs idle (256^3: 4 tiles)
    const Dims& z = p->dims[0];
    if (!p->small && L == 0 && p->opt.small_fused && !(e && e[0] == '1') && p->opt.shard_count == 1 && !p->dist_comm &&
        !p->p2p && z.P >= 1 && z.Q >= 1 && z.N >= 1 && z.Q < (1LL << 30) &&
        ((z.P + 127) / 128) * ((z.N + 127) / 128) < gemm_sm_count() && small_config(1, 1, (int)z.Q, 1, &kc, &g)) {
      p->small = true;
      FMM_CUDA(cudaMalloc(&p->small_M, 16));  // unused: the tiles go straight to C
      FMM_CUDA(cudaMalloc(&p->small_cnt, 16));
    }
  }
  p->setup_sharding();
  p->setup_workspace();
  // compile the streaming/write-once kernels for the 16-byte variant now (NVRTC)
  if (p->L > 0) {
    if (!p->formU.empty()) p->kernel(0, 2);
    if (!p->formV.empty()) p->kernel(1, 2);
    p->kernel(2, 2);
  }
  // size the tables with a dry build (pointer values do not change the table sizes)
  p->build(reinterpret_cast<const double*>(0x100000), std::max<long long>(p->Q, 1), reinterpret_cast<const double*>(0x200000),
           std::max<long long>(p->N, 1), reinterpret_cast<double*>(0x300000), std::max<long long>(p->N, 1), true);
  p->tab_bytes = std::max<size_t>(p->h_tab.size(), 256);
  p->scratch_elems = p->scratch_used;
  if (p->scratch_elems) {
    const size_t bytes = p->scratch_elems * sizeof(double);
    if (p->opt.workspace_limit_bytes && p->ws_bytes + bytes > p->opt.workspace_limit_bytes)
      throw Error(FMM_E_NO_MEMORY, "plan needs " + std::to_string(p->ws_bytes + bytes) +
                                       " workspace bytes with its memory CSE temporaries > limit");
    if (cudaMalloc(reinterpret_cast<void**>(&p->scratch), bytes) != cudaSuccess) {
      cudaGetLastError();
      p->scratch = nullptr;
      throw Error(FMM_E_NO_MEMORY, "cudaMalloc of " + std::to_string(bytes) + " CSE temporary bytes failed");
    }
    p->ws_bytes += bytes;
  }
  for (auto& sl : p->slot) FMM_CUDA(cudaMalloc(&sl.d_tab, p->tab_bytes));
  FMM_CUDA(cudaMallocHost(&p->h_pinned, p->tab_bytes));
  FMM_CUDA(cudaEventCreateWithFlags(&p->upload_done, cudaEventDisableTiming));
  for (auto& e : p->ev) FMM_CUDA(cudaEventCreate(&e));
  if (p->fuse && p->L >= 1) {
    p->ctr_bytes = sizeof(unsigned long long) * (size_t)(2 + 2 * p->nodes_at[p->L - 1] + 4);  // + 4 diagnostics
    FMM_CUDA(cudaMalloc(&p->d_ctr, p->ctr_bytes));
  }
}

#define FMM_CHECK_STATUS(x)                                  \
  do {                                                       \
    const fmm_status_t st_ = (x);                            \
    if (st_ != FMM_OK) throw Error(st_, "internal call failed"); \
  } while (0)

void check_ld(const fmm_plan_t* p, long long lda, long long ldb, long long ldc) {
  // user-orientation requirements (fmm.h)
  if (!p->colmajor) {
    if (lda < std::max<long long>(p->userQ, 1) || ldb < std::max<long long>(p->userN, 1) || ldc < std::max<long long>(p->userN, 1))
      throw Error(FMM_E_SHAPE, "row-major requires lda >= Q, ldb >= Nc, ldc >= Nc");
  } else {
    if (lda < std::max<long long>(p->userP, 1) || ldb < std::max<long long>(p->userQ, 1) || ldc < std::max<long long>(p->userP, 1))
      throw Error(FMM_E_SHAPE, "column-major requires lda >= P, ldb >= Q, ldc >= P");
  }
}

// Enqueue the plan on `stream`; if ev_phase is non-null, record events between phases.
void run(fmm_plan_t* p, const double* A, long long lda, const double* B, long long ldb, double* C, long long ldc,
         cudaStream_t stream, cudaEvent_t* evs) {
  const bool timed = evs != nullptr;
  // a pointer may be null only when its matrix is empty
  if ((!A && p->userP * p->userQ > 0) || (!B && p->userQ * p->userN > 0) || (!C && p->userP * p->userN > 0))
    throw Error(FMM_E_INVALID_ARG, "null matrix pointer");
  check_ld(p, lda, ldb, ldc);
  {  // C must not overlap A or B (fmm.h): compare the byte spans of the three storages
    const bool cm = p->colmajor;
    auto span = [](const double* x, long long rows, long long cols, long long ld) {
      const uintptr_t lo = reinterpret_cast<uintptr_t>(x);
      return std::make_pair(lo, rows > 0 && cols > 0 ? lo + (uintptr_t)(((rows - 1) * ld + cols) * 8) : lo);
    };
    const auto sa = span(A, cm ? p->userQ : p->userP, cm ? p->userP : p->userQ, lda);
    const auto sb = span(B, cm ? p->userN : p->userQ, cm ? p->userQ : p->userN, ldb);
    const auto sc = span(C, cm ? p->userN : p->userP, cm ? p->userP : p->userN, ldc);
    auto overlap = [](std::pair<uintptr_t, uintptr_t> x, std::pair<uintptr_t, uintptr_t> y) {
      return x.first < x.second && y.first < y.second && x.first < y.second && y.first < x.second;
    };
    if (overlap(sc, sa) || overlap(sc, sb)) throw Error(FMM_E_INVALID_ARG, "C must not overlap A or B");
  }
  FMM_CUDA(cudaSetDevice(p->device));
  // a peer-memory plan computes its partial product into the p2p buffer (contiguous, plan
  // orientation) and sums the ranks' partials into the caller's C at the end
  double* const userC = C;
  const long long user_ldc = ldc;
  const long long crows = p->colmajor ? p->userN : p->userP, ccols = p->colmajor ? p->userP : p->userN;
  // push mode (p2p_push, root output): this rank's partial goes straight into its slot of the
  // root's buffer -- the kernels that write C store over peer memory, tile by tile
  const bool push = p->p2p && p->opt.p2p_push && p->dist_root != FMM_DIST_SLABS;
  const long long slot_elems = (crows * ccols + 1) / 2 * 2;  // slots 16-byte aligned
  if (p->p2p) {
    const size_t need = (size_t)(push ? slot_elems * p2p_nranks(p->p2p) : crows * ccols) * 8;
    if (need > p2p_bytes(p->p2p))
      throw Error(FMM_E_SHAPE, push ? "the p2p buffer holds fewer than G partials (p2p_push)" : "the p2p partial buffer is smaller than C");
    C = push ? p2p_peer(p->p2p, p->dist_root) + (size_t)p2p_rank(p->p2p) * slot_elems : p2p_local(p->p2p);
    ldc = std::max<long long>(ccols, 1);
  }
  // row-major orientation: for column-major, C^T = B^T A^T (Prop. 1)
  const double* a = p->colmajor ? B : A;
  const double* b = p->colmajor ? A : B;
  const long long la = p->colmajor ? ldb : lda, lb = p->colmajor ? lda : ldb;
  fmm_plan_s::Slot* sl = nullptr;
  for (auto& c : p->slot)
    if (c.valid && c.A == a && c.B == b && c.C == C && c.lda == la && c.ldb == lb && c.ldc == ldc) sl = &c;
  if (!sl) {
    sl = p->slot[0].used <= p->slot[1].used ? &p->slot[0] : &p->slot[1];
    p->build(a, la, b, lb, C, ldc, false);
    if (p->h_tab.size() > p->tab_bytes) throw Error(FMM_E_INVALID_ARG, "internal: table size grew");
    FMM_CUDA(cudaEventSynchronize(p->upload_done));  // the previous upload has consumed h_pinned
    std::memcpy(p->h_pinned, p->h_tab.data(), p->h_tab.size());
    // stream-ordered: kernels of earlier executes on this stream that read the slot finish first
    FMM_CUDA(cudaMemcpyAsync(sl->d_tab, p->h_pinned, p->h_tab.size(), cudaMemcpyHostToDevice, stream));
    FMM_CUDA(cudaEventRecord(p->upload_done, stream));
    if (sl->gexec) FMM_CUDA(cudaGraphExecDestroy(sl->gexec));
    sl->gexec = nullptr;
    sl->runs = 0;
    sl->valid = true;
    sl->A = a;
    sl->B = b;
    sl->C = C;
    sl->lda = la;
    sl->ldb = lb;
    sl->ldc = ldc;
    sl->launches = p->launches;
  }
  sl->used = ++p->use_clock;
  char* d_tab = sl->d_tab;
  if (timed) FMM_CUDA(cudaEventRecord(evs[0], stream));
  int phase = 0;  // 0 formation, 1 gemm, 2 assembly/strips
  // CUDA-graph replay of a cached slot (option cuda_graphs): captured on the slot's second use,
  // on a private stream, then launched on the caller's stream (kernels only: the table upload
  // happened when the slot was built; fused launches need their counter reset and stay plain)
  bool graphable = p->opt.cuda_graphs && !timed && !p->dist_comm && !p->p2p;
  for (const Launch& ln : sl->launches) graphable &= ln.kind != Launch::FUSED;
  if (graphable && sl->gexec) {
    FMM_CUDA(cudaGraphLaunch(sl->gexec, stream));
    ++sl->runs;
    return;
  }
  const bool capture = graphable && sl->runs >= 1;
  cudaStream_t ls = stream;  // the stream the launches below go to
  if (capture) {
    if (!p->s_cap) FMM_CUDA(cudaStreamCreateWithFlags(&p->s_cap, cudaStreamNonBlocking));
    ls = p->s_cap;
    FMM_CUDA(cudaStreamBeginCapture(ls, cudaStreamCaptureModeThreadLocal));
  }
  struct CaptureGuard {  // a launch that throws mid-capture must not leave the stream capturing
    cudaStream_t s;
    bool on;
    ~CaptureGuard() {
      if (!on) return;
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(s, &g);
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
    }
  } guard{ls, capture};
  // NCCL plans with chunked assembly: a chunk's rows of C are reduced on s_comm right after it
  const bool chunked = p->dist_comm && ccols > 0 && crows > 0 &&
                       std::any_of(sl->launches.begin(), sl->launches.end(), [](const Launch& x) { return !x.reduce_rows.empty(); });
  int nchunk_ev = 0;
  if (chunked) {
    if (crows > 1 && ldc != ccols) throw Error(FMM_E_UNSUPPORTED, "a distributed plan needs a contiguous C");
    if (!p->s_comm) FMM_CUDA(cudaStreamCreateWithFlags(&p->s_comm, cudaStreamNonBlocking));
  }
  int nl = 0;  // profile_launches: events recorded so far
  auto mark = [&](int phase_of_launch, int kind = -1, int level = -1) {
    if (!p->profile_launches) return;
    if ((int)p->ev_l.size() <= nl) {
      cudaEvent_t e;
      FMM_CUDA(cudaEventCreate(&e));
      p->ev_l.push_back(e);
      p->ev_l_phase.push_back(0);
      p->ev_l_kind.push_back(-1);
      p->ev_l_level.push_back(-1);
    }
    p->ev_l_phase[nl] = phase_of_launch;
    p->ev_l_kind[nl] = kind;
    p->ev_l_level[nl] = level;
    FMM_CUDA(cudaEventRecord(p->ev_l[nl++], ls));
  };
  mark(-1);  // start
  auto reduce_after = [&](const Launch& ln) {
    if (!chunked || ln.reduce_rows.empty()) return;
    if ((int)p->ev_chunk.size() <= nchunk_ev) {
      cudaEvent_t e;
      FMM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      p->ev_chunk.push_back(e);
    }
    cudaEvent_t e = p->ev_chunk[nchunk_ev++];
    FMM_CUDA(cudaEventRecord(e, ls));
    FMM_CUDA(cudaStreamWaitEvent(p->s_comm, e, 0));
    dist_reduce_rows(p->dist_comm, p->opt.shard_count, C, crows, ccols, ln.reduce_rows, p->dist_root, p->s_comm);
  };
  // NVTX: one range per launch, named by phase and recursion level (profiling)
  static const char* const kNvtx[] = {"fmm form A", "fmm form B",           "fmm leaf gemm", "fmm assemble", "fmm strips",
                                      "fmm thin",   "fmm fused leaf level", "fmm reduce",    "fmm zero",
                                      "fmm small fused step"};
  static_assert(sizeof(kNvtx) / sizeof(kNvtx[0]) == Launch::SMALL + 1, "one NVTX name per launch kind");
  char nvtx_name[64];
  nvtxRangePushA(p->dist_comm || p->p2p ? "fmm_execute (distributed)" : "fmm_execute");
  struct NvtxPop {
    ~NvtxPop() { nvtxRangePop(); }
  } nvtx_outer;
  for (const Launch& ln : sl->launches) {
    std::snprintf(nvtx_name, sizeof nvtx_name, "%s L%d", kNvtx[(int)ln.kind], ln.level);
    nvtxRangePushA(nvtx_name);
    NvtxPop nvtx_launch;
    if (ln.kind == Launch::REDUCE) {
      reduce_after(ln);
      continue;
    }
    const int ph = (ln.kind == Launch::FORM_A || ln.kind == Launch::FORM_B) ? 0
                   : (ln.kind == Launch::GEMM || ln.kind == Launch::FUSED || ln.kind == Launch::SMALL ||
                      (ln.kind == Launch::SKINNY && ln.level == p->L))
                       ? 1
                       : 2;
    const int prof_phase = ph < 2 ? ph : (ln.kind == Launch::ASSEMBLE || ln.kind == Launch::ZERO) ? 2 : 3;
    if (ln.kind == Launch::SKINNY) {
      const int* ids = reinterpret_cast<const int*>(d_tab + ln.ids_off);
      if (timed && ph != phase) {
        for (int q = phase + 1; q <= ph; ++q) FMM_CUDA(cudaEventRecord(evs[q], stream));
        phase = ph;
      }
      skinny_launch(reinterpret_cast<const GemmTask*>(d_tab + ln.table_off), ids, ln.nrow, ln.max_n, ids + ln.nrow,
                    ln.ncol, ln.max_m, ls, ln.thin_r, ln.thin_c);
      mark(prof_phase, (int)ln.kind, ln.level);
      continue;
    }
    if (timed && ph != phase) {
      for (int q = phase + 1; q <= ph; ++q) FMM_CUDA(cudaEventRecord(evs[q], stream));
      phase = ph;
    }
    const void* tab = d_tab + ln.table_off;
    switch (ln.kind) {
      case Launch::FORM_A:
      case Launch::FORM_B:
      case Launch::ASSEMBLE:
        lincomb_launch(*ln.kern, tab, ln.count, ln.rows, ln.cols, ls);
        break;
      case Launch::SKINNY:
      case Launch::REDUCE:
        break;
      case Launch::SMALL:
        small_launch(ln.small, ls);
        break;
      case Launch::ZERO:
        for (const auto& zb : ln.zero_blocks)
          FMM_CUDA(cudaMemset2DAsync(reinterpret_cast<void*>((uintptr_t)zb[0]), (size_t)zb[1] * 8, 0, (size_t)zb[3] * 8,
                                     (size_t)zb[2], ls));
        break;
      case Launch::FUSED: {
        FusedArgs fa{};
        for (int q = 0; q < ln.nprogs; ++q) {
          fa.node_tab[q] = d_tab + ln.prog_node_off[q];
          fa.node_bytes[q] = ln.prog_node_bytes[q];
          fa.cols[q] = ln.prog_cols[q];
          fa.vec2[q] = ln.prog_vec2[q];
        }
        fa.jobs = reinterpret_cast<const FusedJob*>(d_tab + ln.jobs_off);
        fa.njobs0 = ln.njobs0;
        fa.njobs = ln.njobs;
        fa.ctr = p->d_ctr;
        fa.ready_target = reinterpret_cast<const int*>(d_tab + ln.targets_off);
        fa.tiles_target = fa.ready_target + ln.np;
        fa.np = ln.np;
        fa.gemm_ctas = ln.gemm_ctas;
        FMM_CUDA(cudaMemsetAsync(p->d_ctr, 0, p->ctr_bytes, stream));
        fused_launch(*ln.fk, reinterpret_cast<const GemmTask*>(tab), d_tab + ln.maps_off, ln.count, ln.tiles, ln.uni_tm,
                     ln.uni_tn, fa, stream);
        if (getenv("FMM_FUSED_STATS")) {  // diagnostics (blocking): the kernel's wait / job clock totals
          unsigned long long v[4];
          FMM_CUDA(cudaMemcpyAsync(v, p->d_ctr + 2 + 2 * ln.np, sizeof(v), cudaMemcpyDeviceToHost, stream));
          FMM_CUDA(cudaStreamSynchronize(stream));
          fprintf(stderr, "fused stats (Mcycles summed over threads/warps): ready_wait %.3f tile_wait %.3f jobs_bg %.3f jobs_consumer %.3f\n",
                  v[0] * 1e-6, v[1] * 1e-6, v[2] * 1e-6, v[3] * 1e-6);
        }
        break;
      }
      case Launch::GEMM:
      case Launch::STRIPS:
        if (ln.k3f) {
          K3fArgs ka;
          ka.maps = d_tab + ln.k3f_maps_off;
          ka.count = reinterpret_cast<const int*>(d_tab + ln.k3f_count_off);
          ka.targets = reinterpret_cast<const K3fTarget*>(d_tab + ln.k3f_targets_off);
          gemm_k3f_launch(reinterpret_cast<const GemmTask*>(tab), d_tab + ln.maps_off, ln.count, ln.tiles, ln.uni_tm,
                          ln.uni_tn, ka, ls);
        } else if (ln.tma)
          gemm_tma_launch(reinterpret_cast<const GemmTask*>(tab), d_tab + ln.maps_off, ln.count, ln.tiles, ln.bn,
                          ln.bk, ln.uni_tm, ln.uni_tn, ls, ln.epi);
        else
          gemm_launch(reinterpret_cast<const GemmTask*>(tab), ln.count, ln.tiles, ln.aligned16, ls);
        break;
    }
    mark(prof_phase, (int)ln.kind, ln.level);
    reduce_after(ln);
  }
  if (capture) {
    cudaGraph_t g = nullptr;
    guard.on = false;
    FMM_CUDA(cudaStreamEndCapture(ls, &g));
    const cudaError_t e = cudaGraphInstantiate(&sl->gexec, g, 0);
    cudaGraphDestroy(g);
    FMM_CUDA(e);
    FMM_CUDA(cudaGraphLaunch(sl->gexec, stream));
  }
  ++sl->runs;
  if (timed) {  // phase [3] ends with the last kernel; a combine after it is the caller's next phase
    for (int q = phase + 1; q <= 3; ++q) FMM_CUDA(cudaEventRecord(evs[q], stream));
    phase = 3;
  }
  if (chunked) {  // the caller's stream continues once the last chunk reduce is done
    if ((int)p->ev_chunk.size() <= nchunk_ev) {
      cudaEvent_t e;
      FMM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      p->ev_chunk.push_back(e);
    }
    cudaEvent_t e = p->ev_chunk[nchunk_ev];
    FMM_CUDA(cudaEventRecord(e, p->s_comm));
    FMM_CUDA(cudaStreamWaitEvent(stream, e, 0));
  } else if (p->dist_comm) {  // a7: the partial products of all ranks summed on the root
    const long long rows = crows, cols = ccols;
    if (rows > 1 && ldc != cols) throw Error(FMM_E_UNSUPPORTED, "a distributed plan needs a contiguous C");
    if (rows * cols > 0) {
      if (p->dist_root == FMM_DIST_SLABS) dist_reduce_slabs(p->dist_comm, p->opt.shard_count, C, rows, cols, stream);
      else dist_reduce(p->dist_comm, C, (size_t)rows * cols, p->dist_root, stream);
    }
  }
  if (p->p2p) {  // a7 over peer memory: every partial complete -> pull-reduce -> every read done
    auto bar = [&]() {
      if (p->barrier(p->barrier_ctx) != 0) throw Error(FMM_E_NCCL, "the peer-memory plan's host barrier failed");
    };
    FMM_CUDA(cudaStreamSynchronize(stream));
    bar();
    const int g = p2p_rank(p->p2p), G = p2p_nranks(p->p2p);
    long long r0 = 0, r1 = 0;
    if (p->dist_root == FMM_DIST_SLABS) dist_slab_range(crows, G, g, &r0, &r1);
    else if (p->dist_root == g) r0 = 0, r1 = crows;
    if (push) {  // every partial is in the root's slots: the root sums them locally
      if (p->dist_root == g && crows > 0 && ccols > 0)
        p2p_reduce_slots(p->p2p, slot_elems, crows, ccols, ldc, userC, user_ldc, stream);
    } else if (r1 > r0 && ccols > 0) {
      p2p_reduce_rows(p->p2p, crows, r0, r1, ccols, ldc, userC + r0 * user_ldc, user_ldc, stream);
    }
    FMM_CUDA(cudaStreamSynchronize(stream));
    bar();
  }
  if (p->profile_launches && (p->dist_comm || p->p2p)) {
    if ((int)p->ev_l.size() <= nl) {
      cudaEvent_t e;
      FMM_CUDA(cudaEventCreate(&e));
      p->ev_l.push_back(e);
      p->ev_l_phase.push_back(0);
      p->ev_l_kind.push_back(-1);
      p->ev_l_level.push_back(-1);
    }
    p->ev_l_phase[nl] = 4;
    p->ev_l_kind[nl] = Launch::REDUCE;
    p->ev_l_level[nl] = 0;
    FMM_CUDA(cudaEventRecord(p->ev_l[nl++], stream));
  }
  if (p->profile_launches) p->ev_l_phase.resize(nl);
}

}  // namespace

extern "C" {

void fmm_plan_options_default(fmm_plan_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->layout = FMM_ROW_MAJOR;
  o->strategy = FMM_ADD_STREAMING;
  o->cse = 1;
  o->shard_rank = 0;
  o->shard_count = 1;
  o->workspace_limit_bytes = 0;
  o->peel_align = 1;
  o->fuse_leaf_level = 0;  // within +-2 % of the separate kernels on B200
  o->collapse_levels = 1;
  o->cuda_graphs = 1;
  o->peel_tiles = 0;  // measured: c3 12.60 -> 12.78 ms, c5 258.0 -> 257.3 (R7c)
  o->dist_chunks = 4;
  o->fuse_output = 0;
  o->small_fused = 1;
  o->p2p_push = 0;
}

fmm_status_t fmm_plan_create(const fmm_alg* alg, int64_t P, int64_t Q, int64_t Nc, int levels,
                             const fmm_plan_options* opt, int device, fmm_plan_t** out) {
  FMM_API_BEGIN
  if (!out) throw Error(FMM_E_INVALID_ARG, "null out");
  *out = nullptr;
  std::unique_ptr<fmm_plan_t> p(new fmm_plan_t);
  plan_init(p.get(), alg, P, Q, Nc, levels, opt, device);
  *out = p.release();
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_plan_create_dist(const fmm_alg* alg, int64_t P, int64_t Q, int64_t Nc, int levels,
                                  const fmm_plan_options* opt, fmm_comm* comm, int root, fmm_plan_t** out) {
  FMM_API_BEGIN
  if (!out || !comm) throw Error(FMM_E_INVALID_ARG, "null argument");
  if (root != FMM_DIST_SLABS && (root < 0 || root >= comm_nranks(comm))) throw Error(FMM_E_INVALID_ARG, "bad root");
  *out = nullptr;
  fmm_plan_options o;
  if (opt) o = *opt;
  else fmm_plan_options_default(&o);
  o.shard_rank = comm_rank(comm);
  o.shard_count = comm_nranks(comm);
  std::unique_ptr<fmm_plan_t> p(new fmm_plan_t);
  p->dist_comm = comm_handle(comm);  // before plan_init: its dry build sizes the chunk tables
  p->dist_root = root;
  plan_init(p.get(), alg, P, Q, Nc, levels, &o, comm_device(comm));
  *out = p.release();
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_plan_create_p2p(const fmm_alg* alg, int64_t P, int64_t Q, int64_t Nc, int levels,
                                 const fmm_plan_options* opt, fmm_p2p* p2p, int root, fmm_barrier_fn barrier,
                                 void* barrier_ctx, fmm_plan_t** out) {
  FMM_API_BEGIN
  if (!out || !p2p || !barrier) throw Error(FMM_E_INVALID_ARG, "null argument");
  if (root != FMM_DIST_SLABS && (root < 0 || root >= p2p_nranks(p2p))) throw Error(FMM_E_INVALID_ARG, "bad root");
  if (P < 0 || Nc < 0) throw Error(FMM_E_SHAPE, "negative dimension");
  if ((size_t)P * (size_t)Nc * 8 > p2p_bytes(p2p)) throw Error(FMM_E_SHAPE, "the p2p partial buffer is smaller than P x Nc doubles");
  *out = nullptr;
  fmm_plan_options o;
  if (opt) o = *opt;
  else fmm_plan_options_default(&o);
  o.shard_rank = p2p_rank(p2p);
  o.shard_count = p2p_nranks(p2p);
  std::unique_ptr<fmm_plan_t> p(new fmm_plan_t);
  p->p2p = p2p;
  p->barrier = barrier;
  p->barrier_ctx = barrier_ctx;
  p->dist_root = root;
  plan_init(p.get(), alg, P, Q, Nc, levels, &o, p2p_device(p2p));
  *out = p.release();
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_dist_slab(int64_t P, int64_t Nc, int layout, int nranks, int rank, int64_t* first, int64_t* last) {
  FMM_API_BEGIN
  if (!first || !last) throw Error(FMM_E_INVALID_ARG, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(FMM_E_INVALID_ARG, "bad rank / nranks");
  if (layout != FMM_ROW_MAJOR && layout != FMM_COL_MAJOR) throw Error(FMM_E_INVALID_ARG, "bad layout");
  if (P < 0 || Nc < 0) throw Error(FMM_E_SHAPE, "negative dimension");
  long long r0, r1;
  dist_slab_range(layout == FMM_ROW_MAJOR ? P : Nc, nranks, rank, &r0, &r1);
  *first = r0;
  *last = r1;
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_plan(const fmm_alg* alg, int64_t M, int64_t K, int64_t N, int levels, fmm_plan_t** out) {
  int dev = 0;
  cudaGetDevice(&dev);
  return fmm_plan_create(alg, M, K, N, levels, nullptr, dev, out);
}

fmm_status_t fmm_plan_input_blocks(const fmm_plan_t* p, uint8_t* needA, uint8_t* needB, int64_t core[3], int* need_all) {
  FMM_API_BEGIN
  if (!p || !needA || !needB || !core || !need_all) throw Error(FMM_E_INVALID_ARG, "null argument");
  const fmm_alg* a = p->alg;  // plan orientation (the Prop. 1 transpose for column-major plans)
  const int M = a->M, K = a->K, Nb = a->N, R = a->R;
  std::vector<uint8_t> pa((size_t)M * K, 0), pb((size_t)K * Nb, 0);
  const Dims& d0 = p->dims[0];
  const bool strips = d0.P1 < d0.P || d0.Q1 < d0.Q || d0.N1 < d0.N;
  bool all = p->L < 1 || (strips && p->strip_owner[0][0]);
  if (!all)
    for (int r = 0; r < R; ++r) {
      if (!p->needed[1][r]) continue;
      for (int i = 0; i < M * K; ++i) pa[i] |= a->Ud[(size_t)i * R + r] != 0.0;
      for (int j = 0; j < K * Nb; ++j) pb[j] |= a->Vd[(size_t)j * R + r] != 0.0;
    }
  if (all) std::fill(pa.begin(), pa.end(), 1), std::fill(pb.begin(), pb.end(), 1);
  // back to the caller's orientation: column-major plans multiply B^T A^T with <N,K,M>, so the plan's
  // A block (c, b) is the caller's B block (b, c) and the plan's B block (b, a) the caller's A block (a, b)
  if (!p->colmajor) {
    std::copy(pa.begin(), pa.end(), needA);
    std::copy(pb.begin(), pb.end(), needB);
    core[0] = d0.P1, core[1] = d0.Q1, core[2] = d0.N1;
  } else {
    const int uM = Nb, uN = M;  // the caller's base case is <Nb, K, M> of the plan's <M, K, Nb>
    for (int b = 0; b < K; ++b)
      for (int c = 0; c < uN; ++c) needB[b * uN + c] = pa[c * K + b];
    for (int x = 0; x < uM; ++x)
      for (int b = 0; b < K; ++b) needA[x * K + b] = pb[b * Nb + x];
    core[0] = d0.N1, core[1] = d0.Q1, core[2] = d0.P1;
  }
  *need_all = all ? 1 : 0;
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_plan_workspace_bytes(const fmm_plan_t* p, size_t* bytes) {
  FMM_API_BEGIN
  if (!p || !bytes) throw Error(FMM_E_INVALID_ARG, "null argument");
  *bytes = p->ws_bytes;
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_plan_stats(const fmm_plan_t* p, double out[8]) {
  FMM_API_BEGIN
  if (!p || !out) throw Error(FMM_E_INVALID_ARG, "null argument");
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (const Launch& ln : p->launches) {
    s[0] += ln.flops;
    s[1] += ln.elem_adds;
    s[2] += 8.0 * (ln.elem_reads + ln.elem_writes);
    s[3] += ln.gemm_bytes;
    s[4] += ln.kind == Launch::REDUCE ? 0
            : (ln.kind == Launch::FORM_A || ln.kind == Launch::FORM_B || ln.kind == Launch::ASSEMBLE) && ln.kern
                ? lincomb_steps(*ln.kern)  // pairwise: one launch per chain position
                : 1;
    if (ln.kind == Launch::GEMM || ln.kind == Launch::FUSED || ln.kind == Launch::SMALL ||
        (ln.kind == Launch::SKINNY && ln.level == p->L))
      s[6] += ln.count;
    if (ln.kind == Launch::SKINNY) s[4] += (ln.nrow > 0) + (ln.ncol > 0) - 1;
  }
  s[5] = p->L;
  s[7] = 2.0 * p->userP * p->userQ * (double)p->userN - (double)p->userP * p->userN;
  std::memcpy(out, s, sizeof(s));
  return FMM_OK;
  FMM_API_END
}

}  // extern "C"

// ---- cost model: predicted time of a plan (the paper's cutoff question, Sec. 3.4) -----
// Leaf products: the persistent DMMA kernel's tile schedule (128 x BN tiles from the same width menu,
// wave quantisation over the SMs, a fixed per-tile prologue/epilogue); thin products on the CUDA
// cores; additions: streaming traffic (P:634-636 in bytes) at the addition kernels' measured HBM
// rate; a fixed cost per launch.  Rates are the round-1 B200 measurements.
namespace {
struct CostModel {
  int sms = 148;
  double f_sm = 245e9;          // DMMA flop/s per SM on large tiles (0.97 x 37 TF / 148)
  double add_bw = 6.0e12;       // K1 / K3 streaming kernels, bytes/s
  double thin = 25e9;           // CUDA-core thin-strip flop/s per SM
  double launch = 4e-6;         // seconds per kernel launch
};

double gemm_time(double count, long long m, long long n, long long k, const CostModel& cm) {
  if (count <= 0 || m <= 0 || n <= 0) return 0.0;
  if (k <= 0) return cm.launch;
  if (std::min(m, n) <= 8) return 2.0 * count * m * n * (double)k / (cm.sms * cm.thin) + cm.launch;
  static const int menu[] = {128, 112, 96, 80, 64};
  static const double eff[] = {1.00, 0.998, 0.996, 0.996, 0.993};  // as gemm_choose_bn (round-2 kernel)
  double best = 1e300;
  for (int q = 0; q < 5; ++q) {
    const double tiles = count * (double)((m + 127) / 128) * (double)((n + menu[q] - 1) / menu[q]);
    const double t_tile = 2.0 * 128 * menu[q] * (double)(((k + 15) / 16) * 16 + 32) / (cm.f_sm * eff[q]);
    best = std::min(best, std::ceil(tiles / cm.sms) * t_tile);
  }
  return best + cm.launch;
}

int formed_columns(const std::vector<double>& X, int rows, int R) {
  int f = 0;
  for (int r = 0; r < R; ++r) {
    int nz = 0;
    for (int i = 0; i < rows; ++i) nz += X[(size_t)i * R + r] != 0.0;
    f += nz != 1;
  }
  return f;
}

// seconds; levels beyond the base case are not taken (R10), as in plan_init
// seconds of a plan with the given per-level dims (dims[0..L]) on one B200
double predict_dims(const fmm_alg& a, const std::vector<PlanDims>& dims) {
  const CostModel cm;
  const int M = a.M, K = a.K, Nb = a.N, R = a.R;
  const int L = (int)dims.size() - 1;
  const int fu = formed_columns(a.Ud, M * K, R), fv = formed_columns(a.Vd, K * Nb, R);
  using D = PlanDims;
  // collapsed last two levels (collapse_levels, as plan_init decides it)
  const bool nopeel = L >= 2 && dims[L - 1].P1 == dims[L - 1].P && dims[L - 1].Q1 == dims[L - 1].Q &&
                      dims[L - 1].N1 == dims[L - 1].N;
  const bool small_case = nopeel && M * K <= 4 && K * Nb <= 4 && M * Nb <= 4;
  const char* cf = getenv("FMM_COLLAPSE_FORM");
  const bool collapse = small_case || (nopeel && M * K <= 9 && K * Nb <= 9 && cf && cf[0] == '1');
  const char* wide = getenv("FMM_WIDE_ASM");  // the wide two-level assembly (sec. 6g), on request only
  const bool collapse_asm = small_case || (nopeel && M * Nb <= 16 && wide && wide[0] == '1');
  auto materialized = [&](const std::vector<double>& X, int rows) {
    std::vector<int> sing(R);
    for (int r = 0; r < R; ++r) {
      int nz = 0;
      for (int i = 0; i < rows; ++i) nz += X[(size_t)i * R + r] != 0.0;
      sing[r] = nz == 1;
    }
    int n = 0;
    for (int r1 = 0; r1 < R; ++r1)
      for (int r2 = 0; r2 < R; ++r2) n += !(sing[r1] && sing[r2]);
    return n;
  };
  double nodes = 1, t = 0;
  for (int l = 1; l <= L; ++l) {
    const D& c = dims[l];
    const D& pd = dims[l - 1];
    // formation and assembly of level l (streaming bytes)
    double bytes = 8.0 * nodes *
                   ((double)(M * K + fu) * c.P * c.Q * (fu > 0) + (double)(K * Nb + fv) * c.Q * c.N * (fv > 0) +
                    (double)(R + M * Nb) * c.P * c.N);
    if (collapse && l == L - 1) {
      const D& c2 = dims[L];
      bytes = 8.0 * nodes *
              ((double)(M * K * M * K + materialized(a.Ud, M * K)) * c2.P * c2.Q +
               (double)(K * Nb * K * Nb + materialized(a.Vd, K * Nb)) * c2.Q * c2.N +
               (collapse_asm ? (double)(R * R + M * Nb * M * Nb) * c2.P * c2.N : (double)(R + M * Nb) * c.P * c.N));
    } else if (collapse && l == L) {
      bytes = collapse_asm ? 0 : 8.0 * nodes * (double)(R + M * Nb) * c.P * c.N;  // its assembly only
    } else if (collapse_asm && l == L - 1) {  // its formation as usual; both levels' assembly at once
      const D& c2 = dims[L];
      bytes = 8.0 * nodes *
              ((double)(M * K + fu) * c.P * c.Q * (fu > 0) + (double)(K * Nb + fv) * c.Q * c.N * (fv > 0) +
               (double)(R * R + M * Nb * M * Nb) * c2.P * c2.N);
    } else if (collapse_asm && l == L) {  // its formation only
      bytes = 8.0 * nodes * ((double)(M * K + fu) * c.P * c.Q * (fu > 0) + (double)(K * Nb + fv) * c.Q * c.N * (fv > 0));
    }
    t += bytes / cm.add_bw + (collapse && l == L ? (collapse_asm ? 0.0 : cm.launch) : cm.launch * (1 + (fu > 0) + (fv > 0)));
    // peel strips of the level-(l-1) nodes
    t += gemm_time(nodes, pd.P1, pd.N1, pd.Q - pd.Q1, cm);
    t += gemm_time(nodes, pd.P - pd.P1, pd.N, pd.Q, cm);
    t += gemm_time(nodes, pd.P1, pd.N - pd.N1, pd.Q, cm);
    nodes *= R;
  }
  t += gemm_time(nodes, dims[L].P, dims[L].N, dims[L].Q, cm);
  return t;
}

// the per-level dims of plan_init (R10 effective levels, R7 peeling, R7b alignment peel with the
// default peel_align), then R7c: the tile-aware row peel of the last split when the cost model
// predicts it faster (peel_tiles)
std::vector<PlanDims> plan_dims(const fmm_alg& a, long long P, long long Q, long long N, int levels, bool peel_align,
                                bool peel_tiles, bool* tiled) {
  const int M = a.M, K = a.K, Nb = a.N;
  std::vector<PlanDims> dims;
  PlanDims d{P, Q, N, 0, 0, 0};
  int L = 0;
  while (true) {
    d.P1 = M * (d.P / M);
    d.Q1 = K * (d.Q / K);
    d.N1 = Nb * (d.N / Nb);
    if (peel_align && L < levels) peel_even(d, K, Nb);
    dims.push_back(d);
    if (L == levels || d.P < M || d.Q < K || d.N < Nb) break;
    d = PlanDims{d.P1 / M, d.Q1 / K, d.N1 / Nb, 0, 0, 0};
    ++L;
  }
  if (tiled) *tiled = false;
  // R7c: the leaves' rows run in 128-row GEMM tiles, so r rows cost ceil(r / 128) tiles.  Peeling
  // the remainder r mod 128 of every leaf into the level-(L-1) classical strips leaves 128-aligned
  // leaves; taken only when the cost model says so (the strips are classical work)
  if (peel_tiles && L >= 1 && dims[L].P >= 128 && dims[L].P % 128 != 0) {
    std::vector<PlanDims> alt = dims;
    const long long rt = 128 * (dims[L].P / 128);
    alt[L - 1].P1 = M * rt;
    alt[L].P = rt;
    alt[L].P1 = M * (rt / M);
    if (predict_dims(a, alt) < 0.995 * predict_dims(a, dims)) {
      dims.swap(alt);
      if (tiled) *tiled = true;
    }
  }
  return dims;
}

double predict_seconds(const fmm_alg& a, long long P, long long Q, long long N, int levels, int* used_levels) {
  const std::vector<PlanDims> dims = plan_dims(a, P, Q, N, levels, true, false, nullptr);  // the default options
  if (used_levels) *used_levels = (int)dims.size() - 1;
  return predict_dims(a, dims);
}
}  // namespace

extern "C" {

fmm_status_t fmm_plan_predict(const fmm_alg* alg, int64_t P, int64_t Q, int64_t Nc, int levels, int layout, double* ms,
                              int* used_levels) {
  FMM_API_BEGIN
  if (!alg || !ms) throw Error(FMM_E_INVALID_ARG, "null argument");
  if (P < 0 || Q < 0 || Nc < 0) throw Error(FMM_E_SHAPE, "negative dimension");
  if (levels < 0 || levels > 8) throw Error(FMM_E_UNSUPPORTED, "levels must be in [0, 8]");
  std::unique_ptr<fmm_alg> t;
  const fmm_alg* a = alg;
  long long p = P, n = Nc;
  if (layout == FMM_COL_MAJOR) t.reset(alg_transpose_prop1(*alg)), a = t.get(), p = Nc, n = P;
  *ms = 1e3 * predict_seconds(*a, p, Q, n, levels, used_levels);
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_select(const fmm_alg* const* algs, int nalgs, int64_t P, int64_t Q, int64_t Nc, int max_levels, int layout,
                        int* alg_index, int* perm, int* levels, double* ms) {
  FMM_API_BEGIN
  if ((nalgs > 0 && !algs) || !alg_index || !perm || !levels || !ms) throw Error(FMM_E_INVALID_ARG, "null argument");
  if (P < 0 || Q < 0 || Nc < 0) throw Error(FMM_E_SHAPE, "negative dimension");
  if (max_levels < 0 || max_levels > 8) throw Error(FMM_E_UNSUPPORTED, "max_levels must be in [0, 8]");
  // classical: one DMMA GEMM (levels = 0 of any algorithm)
  const long long p = layout == FMM_COL_MAJOR ? Nc : P, n = layout == FMM_COL_MAJOR ? P : Nc;
  double best = gemm_time(1, p, n, Q, CostModel());
  *alg_index = -1, *perm = 0, *levels = 0;
  for (int i = 0; i < nalgs; ++i) {
    if (!algs[i]) throw Error(FMM_E_INVALID_ARG, "null algorithm in the candidate list");
    for (int q = 0; q < 6; ++q) {
      fmm_alg* pa = nullptr;
      const fmm_status_t st = fmm_alg_permute(algs[i], q, &pa);
      if (st != FMM_OK) return st;
      std::unique_ptr<fmm_alg> own(pa);
      std::unique_ptr<fmm_alg> tr;
      const fmm_alg* a = pa;
      if (layout == FMM_COL_MAJOR) tr.reset(alg_transpose_prop1(*pa)), a = tr.get();
      for (int L = 1; L <= max_levels; ++L) {
        int used = 0;
        const double tt = predict_seconds(*a, p, Q, n, L, &used);
        if (used < L) break;  // deeper levels are not taken
        if (tt < best * (1 - 1e-9)) best = tt, *alg_index = i, *perm = q, *levels = L;
      }
    }
  }
  *ms = 1e3 * best;
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_fused_compile_check(const fmm_alg* alg, int layout, int cse, int bn) {
  return fmm_fused_compile_check_ex(alg, layout, cse, bn, 16, 1);
}

fmm_status_t fmm_fused_compile_check_ex(const fmm_alg* alg, int layout, int cse, int bn, int ks, int mode) {
  FMM_API_BEGIN
  if (!alg) throw Error(FMM_E_INVALID_ARG, "null algorithm");
  if (mode != 1 && mode != 2) throw Error(FMM_E_INVALID_ARG, "mode must be 1 (addition CTAs) or 2 (background)");
  std::unique_ptr<fmm_alg> t;
  const fmm_alg* a = alg;
  if (layout == FMM_COL_MAJOR) t.reset(alg_transpose_prop1(*alg)), a = t.get();
  const int M = a->M, K = a->K, N = a->N, R = a->R;
  std::vector<LincombSpec> specs;
  for (int side = 0; side < 3; ++side) {
    LincombSpec sp;
    sp.strategy = FMM_ADD_STREAMING;
    sp.cse = cse;
    sp.vec = 2;
    if (side < 2) {
      const int rows = side == 0 ? M * K : K * N;
      const auto& X = side == 0 ? a->Ud : a->Vd;
      std::vector<int> form;
      for (int r = 0; r < R; ++r) {
        int nz = 0;
        for (int i = 0; i < rows; ++i) nz += X[(size_t)i * R + r] != 0.0;
        if (nz != 1) form.push_back(r);
      }
      if (form.empty()) continue;
      sp.nin = rows;
      sp.nout = (int)form.size();
      sp.coef.assign((size_t)sp.nin * sp.nout, 0.0);
      for (int o = 0; o < sp.nout; ++o)
        for (int i = 0; i < rows; ++i) sp.coef[(size_t)o * rows + i] = X[(size_t)i * R + form[o]];
    } else {
      sp.nin = R;
      sp.nout = M * N;
      sp.coef.assign((size_t)sp.nin * sp.nout, 0.0);
      for (int k = 0; k < M * N; ++k)
        for (int r = 0; r < R; ++r) sp.coef[(size_t)k * R + r] = a->Wd[(size_t)k * R + r];
    }
    specs.push_back(sp);
  }
  fused_compile(fused_generate(specs, bn, ks, mode == 2));
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_plan_stats_ex2(const fmm_plan_t* p, double* out, int n) {
  FMM_API_BEGIN
  if (!p || !out || n < 0) throw Error(FMM_E_INVALID_ARG, "bad argument");
  double s[19] = {0};
  FMM_CHECK_STATUS(fmm_plan_stats_ex(p, s));
  s[16] = p->k3f ? 1.0 : 0.0;
  s[17] = p->collapse_asm ? 1.0 : 0.0;
  s[18] = p->small ? 1.0 : 0.0;
  std::memcpy(out, s, sizeof(double) * (size_t)std::min(n, 19));
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_plan_stats_ex(const fmm_plan_t* p, double out[16]) {
  FMM_API_BEGIN
  if (!p || !out) throw Error(FMM_E_INVALID_ARG, "null argument");
  double s[16] = {0};
  FMM_CHECK_STATUS(fmm_plan_stats(p, s));
  for (const Launch& ln : p->launches) {
    const double bytes = 8.0 * (ln.elem_reads + ln.elem_writes);
    const bool leaf = ln.kind == Launch::GEMM || ln.kind == Launch::FUSED || ln.kind == Launch::SMALL ||
                      (ln.kind == Launch::SKINNY && ln.level == p->L);
    if (leaf) s[8] += ln.flops;
    if (ln.kind == Launch::FUSED) s[9] += bytes, s[10] += 1;
    if (ln.kind == Launch::FORM_A || ln.kind == Launch::FORM_B) s[11] += bytes;
    if (ln.kind == Launch::ASSEMBLE || ln.kind == Launch::ZERO || (ln.kind == Launch::GEMM && ln.k3f)) s[12] += bytes;
    if (!leaf && (ln.kind == Launch::STRIPS || ln.kind == Launch::SKINNY)) s[13] += ln.flops;
  }
  s[14] = p->collapse ? 1.0 : 0.0;
  s[15] = p->tiled_peel ? 1.0 : 0.0;
  std::memcpy(out, s, sizeof(s));
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_execute(fmm_plan_t* p, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                         int64_t ldc, void* stream) {
  FMM_API_BEGIN
  if (!p) throw Error(FMM_E_INVALID_ARG, "null plan");
  run(p, A, lda, B, ldb, C, ldc, (cudaStream_t)stream, nullptr);
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_exec(fmm_plan_t* p, const double* A, const double* B, double* C) {
  if (!p) return FMM_E_INVALID_ARG;
  if (!p->colmajor)
    return fmm_execute(p, A, std::max<int64_t>(p->userQ, 1), B, std::max<int64_t>(p->userN, 1), C,
                       std::max<int64_t>(p->userN, 1), nullptr);
  return fmm_execute(p, A, std::max<int64_t>(p->userP, 1), B, std::max<int64_t>(p->userQ, 1), C,
                     std::max<int64_t>(p->userP, 1), nullptr);
}

fmm_status_t fmm_execute_timed(fmm_plan_t* p, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                               int64_t ldc, void* stream, float ms[5]) {
  FMM_API_BEGIN
  if (!p || !ms) throw Error(FMM_E_INVALID_ARG, "null argument");
  // plain launches (no graph) with an event after each one; every launch's time goes to its phase
  p->profile_launches = true;
  struct Off {
    fmm_plan_t* p;
    ~Off() { p->profile_launches = false; }
  } off{p};
  run(p, A, lda, B, ldb, C, ldc, (cudaStream_t)stream, p->ev);
  FMM_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  float acc[5] = {0, 0, 0, 0, 0};
  for (size_t q = 1; q < p->ev_l_phase.size(); ++q) {
    float t = 0;
    FMM_CUDA(cudaEventElapsedTime(&t, p->ev_l[q - 1], p->ev_l[q]));
    const int ph = p->ev_l_phase[q];
    if (ph >= 0 && ph < 5) acc[ph] += t;
  }
  ms[0] = acc[0];
  ms[1] = acc[1];
  ms[2] = acc[2];
  ms[3] = acc[3];
  float total = 0;
  if (p->ev_l_phase.size() > 1) FMM_CUDA(cudaEventElapsedTime(&total, p->ev_l[0], p->ev_l[p->ev_l_phase.size() - 1]));
  ms[4] = total;
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_execute_profile(fmm_plan_t* p, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                                 int64_t ldc, void* stream, int max, int* kind, int* level, float* ms, int* n) {
  FMM_API_BEGIN
  if (!p || !n || max < 0 || (max > 0 && (!kind || !level || !ms))) throw Error(FMM_E_INVALID_ARG, "bad argument");
  p->profile_launches = true;
  struct Off {
    fmm_plan_t* p;
    ~Off() { p->profile_launches = false; }
  } off{p};
  run(p, A, lda, B, ldb, C, ldc, (cudaStream_t)stream, p->ev);
  FMM_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  const int cnt = (int)p->ev_l_phase.size() - 1;
  *n = std::max(cnt, 0);
  for (int q = 0; q < std::min(cnt, max); ++q) {
    float t = 0;
    FMM_CUDA(cudaEventElapsedTime(&t, p->ev_l[q], p->ev_l[q + 1]));
    ms[q] = t;
    kind[q] = p->ev_l_kind[q + 1];
    level[q] = p->ev_l_level[q + 1];
  }
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_execute_events(fmm_plan_t* p, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                                int64_t ldc, void* stream, void* events[4]) {
  FMM_API_BEGIN
  if (!p || !events) throw Error(FMM_E_INVALID_ARG, "null argument");
  for (int q = 0; q < 4; ++q)
    if (!events[q]) throw Error(FMM_E_INVALID_ARG, "null event");
  run(p, A, lda, B, ldb, C, ldc, (cudaStream_t)stream, reinterpret_cast<cudaEvent_t*>(events));
  return FMM_OK;
  FMM_API_END
}

// Host-buffer execution, pipelined: iteration i uses staging set b = i % 2.  The copy-in stream
// waits until compute i-2 has finished reading set b; compute (on `stream`) waits for copy-in i
// and for copy-out i-2 (which reads sC[b]); copy-out i waits for compute i.  Consecutive calls
// therefore overlap H2D of the next problem, compute, and D2H of the previous one (PCIe is full
// duplex).  Host buffers must stay valid (and, for overlap, be pinned) until fmm_sync.
static void host_async(fmm_plan_t* p, const double* A, long long lda, const double* B, long long ldb, double* C,
                       long long ldc, cudaStream_t s) {
  if (!A || !B || !C) throw Error(FMM_E_INVALID_ARG, "null argument");
  check_ld(p, lda, ldb, ldc);
  FMM_CUDA(cudaSetDevice(p->device));
  const long long P = p->userP, Q = p->userQ, N = p->userN;
  const bool cm = p->colmajor;
  // (rows, cols) of the storage: row-major P x Q is P rows of Q; column-major is Q "rows" of P
  const long long aR = cm ? Q : P, aC = cm ? P : Q, bR = cm ? N : Q, bC = cm ? Q : N, cR = cm ? N : P, cC = cm ? P : N;
  if (!p->s_in) {
    FMM_CUDA(cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking));
    FMM_CUDA(cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      FMM_CUDA(cudaEventCreateWithFlags(&p->ev_in[b], cudaEventDisableTiming));
      FMM_CUDA(cudaEventCreateWithFlags(&p->ev_comp[b], cudaEventDisableTiming));
      FMM_CUDA(cudaEventCreateWithFlags(&p->ev_out[b], cudaEventDisableTiming));
    }
  }
  const int b = (int)(p->host_iter++ & 1);
  if (!p->sA[0]) {  // both staging sets at once: a cudaMalloc later would stall the pipeline
    for (int q = 0; q < 2; ++q) {
      FMM_CUDA(cudaMalloc(&p->sA[q], std::max<size_t>(8, (size_t)aR * aC * 8)));
      FMM_CUDA(cudaMalloc(&p->sB[q], std::max<size_t>(8, (size_t)bR * bC * 8)));
      FMM_CUDA(cudaMalloc(&p->sC[q], std::max<size_t>(8, (size_t)cR * cC * 8)));
    }
  }

  // copy in, once compute i-2 has released set b
  FMM_CUDA(cudaStreamWaitEvent(p->s_in, p->ev_comp[b], 0));
  if (aR && aC) FMM_CUDA(cudaMemcpy2DAsync(p->sA[b], aC * 8, A, lda * 8, aC * 8, aR, cudaMemcpyHostToDevice, p->s_in));
  if (bR && bC) FMM_CUDA(cudaMemcpy2DAsync(p->sB[b], bC * 8, B, ldb * 8, bC * 8, bR, cudaMemcpyHostToDevice, p->s_in));
  FMM_CUDA(cudaEventRecord(p->ev_in[b], p->s_in));
  // compute
  FMM_CUDA(cudaStreamWaitEvent(s, p->ev_in[b], 0));
  FMM_CUDA(cudaStreamWaitEvent(s, p->ev_out[b], 0));
  run(p, p->sA[b], std::max<long long>(aC, 1), p->sB[b], std::max<long long>(bC, 1), p->sC[b], std::max<long long>(cC, 1),
      s, nullptr);
  FMM_CUDA(cudaEventRecord(p->ev_comp[b], s));
  // copy out
  FMM_CUDA(cudaStreamWaitEvent(p->s_out, p->ev_comp[b], 0));
  if (cR && cC) FMM_CUDA(cudaMemcpy2DAsync(C, ldc * 8, p->sC[b], cC * 8, cC * 8, cR, cudaMemcpyDeviceToHost, p->s_out));
  FMM_CUDA(cudaEventRecord(p->ev_out[b], p->s_out));
}

fmm_status_t fmm_execute_host_async(fmm_plan_t* p, const double* A, int64_t lda, const double* B, int64_t ldb,
                                    double* C, int64_t ldc, void* stream) {
  FMM_API_BEGIN
  if (!p) throw Error(FMM_E_INVALID_ARG, "null plan");
  host_async(p, A, lda, B, ldb, C, ldc, (cudaStream_t)stream);
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_execute_host(fmm_plan_t* p, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                              int64_t ldc, void* stream) {
  FMM_API_BEGIN
  if (!p) throw Error(FMM_E_INVALID_ARG, "null plan");
  host_async(p, A, lda, B, ldb, C, ldc, (cudaStream_t)stream);
  FMM_CUDA(cudaStreamSynchronize(p->s_out));
  FMM_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_sync(fmm_plan_t* p) {
  FMM_API_BEGIN
  if (!p) throw Error(FMM_E_INVALID_ARG, "null plan");
  FMM_CUDA(cudaSetDevice(p->device));
  FMM_CUDA(cudaDeviceSynchronize());
  FMM_CUDA(cudaGetLastError());
  return FMM_OK;
  FMM_API_END
}

void fmm_plan_destroy(fmm_plan_t* p) { delete p; }

fmm_status_t fmm_dgemm(int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda, const double* B,
                       int64_t ldb, double beta, double* C, int64_t ldc, void* stream) {
  FMM_API_BEGIN
  if (m < 0 || n < 0 || k < 0) throw Error(FMM_E_SHAPE, "negative dimension");
  if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX) throw Error(FMM_E_UNSUPPORTED, "dimension above 2^31-1");
  if (m == 0 || n == 0) return FMM_OK;
  if (!A || !B || !C) throw Error(FMM_E_INVALID_ARG, "null matrix pointer");
  if (lda < std::max<int64_t>(k, 1) || ldb < n || ldc < n) throw Error(FMM_E_SHAPE, "leading dimension too small");
  std::vector<GemmTask> t(1);
  t[0].A = A;
  t[0].B = B;
  t[0].C = C;
  t[0].lda = lda;
  t[0].ldb = ldb;
  t[0].ldc = ldc;
  t[0].m = (int)m;
  t[0].n = (int)n;
  t[0].k = (int)k;
  t[0].alpha = alpha;
  t[0].beta = beta;
  cudaStream_t s = (cudaStream_t)stream;
  // the task descriptor (and its tensor maps) go through a stream-ordered upload
  const bool tma = gemm_tma_eligible(t) && !(getenv("FMM_NO_TMA") && getenv("FMM_NO_TMA")[0] == '1');
  const int bn = tma ? gemm_choose_bn(t) : 128;
  int bk = tma ? gemm_choose_bk(t) : 16;
  const int epi = tma ? gemm_choose_epi(t, bn, &bk) : 0;
  const long long tiles = gemm_prepare(t, 128, bn);
  alignas(128) char buf[1024];
  std::memcpy(buf, t.data(), sizeof(GemmTask));
  if (tma) gemm_tma_maps(t, buf + 512, bk);
  // a stream-ordered descriptor per call: calls on different streams never share one
  GemmTask* d_task = nullptr;
  FMM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_task), sizeof(buf), s));
  FMM_CUDA(cudaMemcpyAsync(d_task, buf, sizeof(buf), cudaMemcpyHostToDevice, s));
  if (tma)
    gemm_tma_launch(d_task, reinterpret_cast<char*>(d_task) + 512, 1, tiles, bn, bk, t[0].tiles_m, t[0].tiles_n, s, epi);
  else
    gemm_launch(d_task, 1, tiles, gemm_tasks_aligned16(t), s);
  FMM_CUDA(cudaFreeAsync(d_task, s));
  return FMM_OK;
  FMM_API_END
}

}  // extern "C"
