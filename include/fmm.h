/*
 * fmm.h — C ABI of the B200-native recursive fast matrix multiplication library (libfmm.so).
 *
 * The method (arXiv 1409.2908, Benson & Ballard; PAPER.md cited as P:<line>): C = A*B computed by
 * a bilinear <M,K,N;R> base-case algorithm given as coefficient matrices (U,V,W) (Sec. 2.2,
 * P:295-331, Eq. lowrank), applied for L recursive steps (Sec. 2.1; Sec. 3.1):
 *   S_r = sum_i u_ir A_i,  T_r = sum_j v_jr B_j,  M_r = S_r * T_r (recursively),  C_k = sum_r w_kr M_r
 * with dynamic peeling of non-divisible dimensions at every level (Sec. 3.5).
 *
 * Conventions shared by every entry point
 *  - Every function returns fmm_status_t; no C++ exception crosses the ABI.  On failure a
 *    human-readable message is available from fmm_last_error() (thread-local, valid until the
 *    next fmm_* call on the same thread).
 *  - Block numbering follows the paper's row-major vectorisation: A-block (a,b) of the
 *    M x K block grid is row a*K+b of U; B-block (b,c) is row b*N+c of V; C-block (a,c) is row
 *    a*N+c of W.  Matrices U (MK x R), V (KN x R), W (MN x R) are passed row-major.
 *  - All matrix data is IEEE binary64.  Leading dimensions are in elements.
 *  - Device pointers passed to fmm_execute are owned by the caller and must live on the plan's
 *    device; the library never allocates or frees caller buffers.  A plan owns its workspace.
 *  - Arguments are validated before any device work; invalid ones return FMM_E_INVALID_ARG or
 *    FMM_E_SHAPE and leave device state untouched.
 *  - There is no CPU fallback: every arithmetic step of fmm_execute runs in this library's
 *    sm_100a kernels.
 */
#ifndef FMM_H
#define FMM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FMM_OK = 0,
  FMM_E_INVALID_ARG = 1,   /* null pointer, negative size, bad option value */
  FMM_E_NOT_EXACT = 2,     /* (U,V,W) fails the Brent equations */
  FMM_E_SHAPE = 3,         /* non-conformable dimensions or too-small leading dimensions */
  FMM_E_NO_MEMORY = 4,     /* workspace allocation failed or exceeds workspace_limit_bytes */
  FMM_E_CUDA = 5,          /* a CUDA runtime / NVRTC error; message has the CUDA string */
  FMM_E_NCCL = 6,          /* reserved for communicator errors */
  FMM_E_UNSUPPORTED = 7,   /* e.g. APA (lambda) algorithms, too many recursion levels */
  FMM_E_PARSE = 8          /* algorithm file syntax error; message names the line */
} fmm_status_t;

typedef struct fmm_alg_s fmm_alg;   /* immutable after creation; safe to share between threads */
typedef struct fmm_plan_s fmm_plan_t; /* owns its workspace; one fmm_execute in flight per plan */
typedef struct fmm_comm_s fmm_comm;   /* an NCCL communicator, one rank per process and GPU */

typedef enum { FMM_ROW_MAJOR = 0, FMM_COL_MAJOR = 1 } fmm_layout;

/* Addition-chain implementations (Sec. 3.2).  STREAMING: one kernel per phase reads
   every input block once and writes every formed S_r / T_r (or C_k) once.
   WRITE_ONCE: one output stream per S_r / T_r / C_k, each reading the blocks of its chain
   (P:628-632).  PAIRWISE: the paper's daxpy chains (footnote): per output, a copy
   of the first term then one y <- y + c x pass per further term, i.e. one launch per chain
   position, each reading two blocks and writing one.  Kept for the Fig. 2 study; all
   three round identically (ascending-index chains) when cse = 0. */
typedef enum { FMM_ADD_STREAMING = 0, FMM_ADD_WRITE_ONCE = 1, FMM_ADD_PAIRWISE = 2 } fmm_add_strategy;

typedef struct {
  int layout;               /* fmm_layout of A, B and C (all three share it) */
  int strategy;             /* fmm_add_strategy */
  int cse;                  /* 1: greedy length-two common-subexpression elimination (Sec. 3.3,
                               P:662-720).  Streaming keeps the temporaries in registers;
                               write-once and pairwise write each one to memory once per node
                               (its own launch) and read it in the chains, with the
                               temporaries in a workspace arena counted by
                               fmm_plan_workspace_bytes (each has its node's input leading
                               dimension, so it can exceed the S_r / T_r storage).  0: every chain is summed in ascending
                               index order (bit-identical to the oracle's order). */
  int shard_rank;           /* multi-GPU leaf sharding (Sec. 4.3 HYBRID arithmetic, P:823-829,
                               with GPUs in place of threads): this plan computes the partial
                               product of its share of the R^L leaves; summing the C of all
                               shard_count plans gives A*B.  0 / 1 for a single GPU. */
  int shard_count;
  size_t workspace_limit_bytes; /* 0 = no limit */
  int peel_align;           /* 1: when the paper's core N' = N floor(Nc/N) gives an odd column-block
                               width, peel to N' = 2N floor(Nc/(2N)) instead (one extra column
                               block in the classical strip), and likewise Q' = 2K floor(Q/(2K))
                               for an odd A column-block width, so every sub-block view is 16-byte
                               aligned and TMA / 16-byte vector paths apply (R7b).
                               0: the paper's minimal peeling everywhere. */
  int fuse_leaf_level;      /* 1: run the last level's formation (S_r, T_r of the leaves), the leaf
                               products and the last level's assembly C_k = sum_r w_kr M_r as ONE
                               cooperative persistent launch: CTAs on some SMs run the DMMA leaf
                               tiles, CTAs on the other SMs run the same generated addition chains
                               as the separate kernels, synchronised per parent node through device
                               counters (bitwise equal to the separate kernels).
                               Streaming strategy only; where collapse_levels applies the collapsed
                               kernels run instead.  Needs TMA-eligible leaf views and no thin
                               leaves, else the plan silently runs the separate kernels.
                               2: the same launch in background mode: every CTA runs leaf tiles
                               and the producer warpgroup's three idle warps run the addition
                               jobs (bitwise equal as well; takes precedence over collapse_levels;
                               measured slower than the separate kernels on every config,
                               DESIGN.md sec. 6b).  Needs 256 bytes of shared memory per job
                               input and producer warp beside the GEMM ring, else separate kernels.
                               0: separate formation / GEMM / assembly launches. */
  int shard_mode;           /* with shard_count > 1: 0 = leaf-level HYBRID sharding (the default:
                               balanced to one leaf row); 1 = the top-level products r1 in contiguous
                               balanced ranges (SURVEY 8(e) mode (i): a rank needs only the A / B
                               blocks of its r1, but R mod G makes it uneven) */
  int collapse_levels;      /* 1: evaluate the last two recursion levels' formation and assembly in
                               one streaming pass each (the level-(L-1) S_r, T_r and M_r are never
                               written to HBM: DESIGN.md sec. 6c), where it applies: streaming,
                               L >= 2, a base case with MK, KN, MN <= 4, no peeling at level L-1.
                               (With the environment variable FMM_WIDE_ASM=1, also the assembly
                               alone for base cases up to MN <= 16, no fused leaf level: DESIGN.md
                               sec. 6g; measured slower than the separate levels, so off.)
                               The chains are the oracle's two levels exactly (CSE is not used
                               there).  0: one level per launch. */
  int cuda_graphs;          /* 1: the second and later fmm_execute calls with the same A/B/C
                               pointers and leading dimensions replay the plan's launch sequence
                               as one CUDA graph (captured once per cached pointer set), which
                               removes the per-launch host overhead.  Not used for distributed,
                               fused or timed executes.  0: plain launches every time. */
  int peel_tiles;           /* 1: when the leaves' row count r is not a multiple of the GEMM's 128-row
                               tile, peel r mod 128 rows of every leaf into the last split's
                               classical strips instead, if the cost model predicts that faster
                               (R7c; measured slower on c3, so off by default).  Exact
                               either way.  0 (default): the paper's minimal peeling of rows. */
  int dist_chunks;          /* NCCL distributed plans (fmm_plan_create_dist): the launch that writes
                               C (the level-1 assembly, C_k = sum_r w_kr M_r) runs as this
                               many row chunks, and each chunk's rows of C are reduced on a library
                               communication stream as soon as the chunk is written, so the
                               reduce of chunk j overlaps the assembly of chunk j + 1.  Applies
                               when that launch is one streaming assembly and the top level has no
                               K peel (its rank-update strip would touch C after the assembly);
                               otherwise, and with 0 or 1, one reduce of the whole C at the end.
                               Default 4.  Ignored by single-GPU and peer-memory plans. */
  int fuse_output;          /* 1: K3f -- the last level's output step C_k = sum_r w_kr M_r
                               fused into the leaf GEMM's epilogue: every leaf tile is staged in
                               shared memory and reduce-added by TMA (cp.reduce.async.bulk.tensor,
                               fp64 add in L2) into each level-(L-1) output block its W column
                               touches, so the leaf products M_r are never written or read back and
                               the level-L assembly launch disappears (the target blocks are zeroed
                               first).  The summation order of those adds is not fixed, so results
                               can differ from run to run by rounding (within the tolerances; exact
                               on integer inputs).  Applies when W has only 0 / +-1 entries and
                               MN <= 16, one shard, no fused leaf level; it replaces the collapsed
                               last two levels.  0 (default): separate assembly kernels. */
  int small_fused;          /* 1 (default): a one-level streaming plan (after the cutoff, levels = 1)
                               with no peeling at the top level, one shard, base case MK, KN, MN <= 64 and
                               R <= 128, whose leaf products would give the leaf GEMM fewer 128-row
                               tiles than the GPU has SMs, runs the whole step as ONE launch: a
                               CTA per (32 x 32 leaf tile, product r) forms its S_r rows and T_r
                               columns from A and B in shared memory, multiplies them on the FP64
                               tensor pipe, and the last CTA of each tile forms C_k = sum_r w_kr M_r
                               in ascending r.  Below the paper's cutoff
                               (Sec. 3.4) the separate launches cost more than the
                               arithmetic.  0: the separate launches. */
  int p2p_push;             /* peer-memory plans (fmm_plan_create_p2p) with a root rank: 1 = the
                               launches that write C (the top-level assembly, the top-level peel
                               strips) store this rank's partial straight into slot `rank` of the
                               root's fmm_p2p buffer over peer memory (NVLink stores), so the
                               transfer overlaps the assembly tile by tile; after a host barrier
                               the root sums its G slots in rank order into C.  Every rank's
                               buffer must then hold G partials (G x C, each slot rounded up to
                               16 bytes).  0 (default): each rank writes its partial locally and the
                               root pulls them (the fmm_p2p_reduce kernel).  Slab output always
                               pulls. */
} fmm_plan_options;

/* Fill *opt with the defaults: row-major, streaming, cse = 1, shard 0 of 1, no limit,
   peel_align = 1, fuse_leaf_level = 0, collapse_levels = 1, cuda_graphs = 1, peel_tiles = 0,
   dist_chunks = 4, fuse_output = 0, small_fused = 1, p2p_push = 0. */
void fmm_plan_options_default(fmm_plan_options* opt);

/* ---- algorithms ------------------------------------------------------------------------- */

/* Create an algorithm for base case <M,K,N> of rank R from exact rational coefficients
   num/den (den > 0).  U_num/U_den are MK x R row-major, V_* KN x R, W_* MN x R.
   The Brent equations sum_r u_ir v_jr w_kr = T_ijk, with T the matmul tensor of
   P:412-421, are verified EXACTLY in 128-bit rational arithmetic over all (MK)(KN)(MN)
   triples; any violation returns FMM_E_NOT_EXACT and *out is left NULL.
   Limits: 1 <= M,K,N <= 16, 1 <= R <= 4096.  Host only; no device work. */
fmm_status_t fmm_alg_create(int M, int K, int N, int R,
                            const int64_t* U_num, const int64_t* U_den,
                            const int64_t* V_num, const int64_t* V_den,
                            const int64_t* W_num, const int64_t* W_den, fmm_alg** out);

/* Load the text format of SPEC S:190: '#' comments; a header line "M K N R exact"; MK rows of
   R entries (U), a blank line, KN rows (V), a blank line, MN rows (W).  Entries are integers or
   rationals p/q.  Syntax errors return FMM_E_PARSE with the 1-based line number in the
   message; APA files ("apa") return FMM_E_UNSUPPORTED; then validates as fmm_alg_create. */
fmm_status_t fmm_alg_load(const char* path, fmm_alg** out);

/* Equivalent algorithm for a permuted base case (Props. 1-2, exact; re-validated):
   perm 0 <M,K,N> (copy), 1 <N,K,M> (Prop. 1), 2 <N,M,K> (Prop. 2), 3 <K,N,M> (Prop. 2 twice),
   4 <K,M,N> (Prop. 1 after Prop. 2), 5 <M,N,K> (Prop. 1 after Prop. 2 twice).  Host only; the
   caller owns *out (fmm_alg_destroy). */
fmm_status_t fmm_alg_permute(const fmm_alg* alg, int perm, fmm_alg** out);

/* Query shape and sparsity: dims[0..3] = M,K,N,R; nnz[0..2] = nnz(U), nnz(V), nnz(W). */
fmm_status_t fmm_alg_info(const fmm_alg* alg, int dims[4], int nnz[3]);
void fmm_alg_destroy(fmm_alg* alg);

/* ---- plans ------------------------------------------------------------------------------ */

/* Plan C (P x Nc) = A (P x Q) * B (Q x Nc) with `levels` recursive steps (0 = one classical
   DMMA GEMM; -1 = the fastest levels <= 4 by the cost model of fmm_plan_predict, the paper's
   cutoff question, Sec. 3.4).  The recursion stops early at a level whose sub-problem is smaller than the base
   case (reading R10/R18 of DESIGN.md).  Column-major problems are planned through the
   transposed algorithm of Prop. 1: a column-major P x Q array is the row-major
   Q x P array of its transpose, so C^T = B^T A^T runs with <N,K,M> and no data moves.
   Allocates the workspace on `device` with cudaMalloc; returns FMM_E_NO_MEMORY if that fails
   or exceeds opt->workspace_limit_bytes (the message states the bytes needed: BFS execution
   keeps every level's S_r, T_r and M_r resident, R/(MN) times the output per step).
   Compiles the plan's addition kernels (NVRTC, sm_100a) on first use of an algorithm/variant.
   opt may be NULL (defaults). */
fmm_status_t fmm_plan_create(const fmm_alg* alg, int64_t P, int64_t Q, int64_t Nc, int levels,
                             const fmm_plan_options* opt, int device, fmm_plan_t** out);

/* ---- multi-GPU (not in the paper, P:1126 future work) --------------------------
   One process per GPU.  Rank 0 calls fmm_nccl_unique_id and shares the 128 bytes with every rank
   (e.g. torch.distributed.broadcast_object_list); every rank then calls fmm_comm_create on its
   own GPU.  NCCL is loaded at run time (libnccl.so.2); FMM_E_NCCL if it is unavailable. */
fmm_status_t fmm_nccl_unique_id(unsigned char id[128]);
fmm_status_t fmm_comm_create(const unsigned char id[128], int nranks, int rank, int device, fmm_comm** out);
fmm_status_t fmm_comm_info(const fmm_comm* comm, int* nranks, int* rank);
void fmm_comm_destroy(fmm_comm* comm);  /* after every plan using it is destroyed */

/* A distributed plan: rank `rank` of `nranks` computes its HYBRID share of the R^L leaves (Sec. 4.3
   arithmetic, with GPUs in place of threads: opt->shard_rank / shard_count are set from
   the communicator) into a partial C, and fmm_execute ends with one in-place NCCL sum-reduce of C
   to `root` on the execute's stream (the C_k combination is linear in the partials).  C must be
   contiguous (ldc = Nc row-major, ldc = P column-major) on every rank, else FMM_E_UNSUPPORTED at
   execute.  The result is complete on `root` only.  The plan keeps `comm` (not owned).
   root = FMM_DIST_SLABS instead gives slab-distributed output (reduce-scatter): the
   contiguous C is cut along its outer storage dimension (rows of C when row-major, columns when
   column-major) into nranks slabs as even as integers allow (fmm_dist_slab), and slab g is summed
   onto rank g -- one grouped set of ncclReduce calls, the same bytes sent as the single reduce.
   Outside its own slab a rank's C holds its partial product. */
#define FMM_DIST_SLABS (-1)
fmm_status_t fmm_plan_create_dist(const fmm_alg* alg, int64_t P, int64_t Q, int64_t Nc, int levels,
                                  const fmm_plan_options* opt, fmm_comm* comm, int root, fmm_plan_t** out);
/* ---- the combine over peer memory (no NCCL in the data path) -------------
   One process per GPU.  Each rank owns a partial-product buffer of `bytes` (cudaMalloc, returned in
   *local): pass it as C to fmm_execute of its shard plan.  Ranks exchange the 64-byte CUDA IPC
   handles of their buffers (fmm_p2p_handle; e.g. torch.distributed all_gather_object) and map
   every peer's with fmm_p2p_open (over NVLink / NVSwitch between GPUs).  fmm_p2p_reduce_slab then
   runs ONE kernel on `stream` that reads the slab of every rank's partial that this rank owns
   (fmm_dist_slab's split of the `outer` dimension; rows of `inner` doubles, leading dimension
   `ld` in the partials) and writes their sum, ranks in ascending order (deterministic), to `out`
   (row r of the slab at out + r * ldo).  Ordering is the caller's: every partial complete before
   any rank reduces, every reduce complete before the next fmm_execute overwrites a partial (e.g.
   stream synchronise + barrier).  At most 16 ranks. */
typedef struct fmm_p2p_s fmm_p2p;
fmm_status_t fmm_p2p_create(int nranks, int rank, int device, size_t bytes, fmm_p2p** out, double** local);
fmm_status_t fmm_p2p_handle(const fmm_p2p* p, unsigned char handle[64]);
fmm_status_t fmm_p2p_open(fmm_p2p* p, const unsigned char* handles /* nranks x 64 bytes */);
fmm_status_t fmm_p2p_reduce_slab(fmm_p2p* p, int64_t outer, int64_t inner, int64_t ld, double* out, int64_t ldo,
                                 void* stream);
void fmm_p2p_destroy(fmm_p2p* p);

/* A distributed plan whose combine runs over peer memory INSIDE fmm_execute (no NCCL in the data
   path): rank p2p->rank of p2p->nranks computes its HYBRID leaf share (as fmm_plan_create_dist) into
   the p2p object's partial buffer, which must hold 8 * P * Nc bytes; then, within the same
   fmm_execute: the stream is synchronised, `barrier(barrier_ctx)` is called (every rank's partial is
   complete), this rank pulls and sums its part of every rank's partial with one kernel
   (fmm_p2p_reduce_slab's kernel, ranks in ascending order) into the caller's C with the caller's
   ldc, the stream is synchronised again and `barrier` is called a second time (no partial is
   overwritten while a peer still reads it).  So fmm_execute of such a plan is BLOCKING.
   root >= 0: rank `root` receives the whole C and the other ranks leave their C untouched;
   root = FMM_DIST_SLABS: every rank receives its fmm_dist_slab slab of C (rows of C when
   row-major, columns when column-major), the rest of its C untouched.
   `barrier` is a host barrier over the same ranks (e.g. torch.distributed.barrier through a
   callback); it returns 0 on success, anything else fails the execute with FMM_E_NCCL.  The plan
   keeps `p2p` (not owned; destroy the plan first).  CUDA graphs are not used for these plans. */
typedef int (*fmm_barrier_fn)(void* ctx);
fmm_status_t fmm_plan_create_p2p(const fmm_alg* alg, int64_t P, int64_t Q, int64_t Nc, int levels,
                                 const fmm_plan_options* opt, fmm_p2p* p2p, int root, fmm_barrier_fn barrier,
                                 void* barrier_ctx, fmm_plan_t** out);

/* The slab of C that rank `rank` of `nranks` holds after a FMM_DIST_SLABS execute: rows
   [*first, *last) of C (row-major) or columns [*first, *last) (column-major).  Host only. */
fmm_status_t fmm_dist_slab(int64_t P, int64_t Nc, int layout, int nranks, int rank, int64_t* first, int64_t* last);

/* Which top-level blocks of A and B this plan reads (host only): a sharded plan (leaf or top-level
   mode) forms only the level-1 S_r / T_r of the products it owns, so it reads A-block (a, b) only if
   u_{(a,b) r} != 0 for one of them (likewise B).  needA has M*K entries (row a*K + b of the caller's
   base case <M,K,N>), needB K*N; core = {P', Q', N'}, the block grid's extent (the blocks are
   P'/M x Q'/K and Q'/K x N'/N); *need_all = 1 when the plan also reads the peeled edges (it owns the
   top-level peel strips) or has no recursion, i.e. all of A and B.  Used to send each rank only
   the input blocks it reads. */
fmm_status_t fmm_plan_input_blocks(const fmm_plan_t* plan, uint8_t* needA, uint8_t* needB, int64_t core[3],
                                   int* need_all);

/* Workspace bytes held by the plan. */
fmm_status_t fmm_plan_workspace_bytes(const fmm_plan_t* plan, size_t* bytes);

/* Predicted work of one fmm_execute, per phase, from the plan's own chain/kernel structure:
   [0] leaf GEMM flops (2 m n k per leaf product and peel strip)
   [1] addition flops (one per add/sub in the emitted chains)
   [2] addition-kernel algorithmic HBM bytes (8 B per element read or written by the
       formation and assembly kernels, Sec. 3.2 counts P:638-653 in bytes)
   [3] leaf GEMM operand/result bytes at one read of S, T and one write of M per leaf
   [4] number of kernel launches per execute
   [5] effective levels used
   [6] number of leaf products computed by this plan (its shard)
   [7] the paper's effective-GFLOPS numerator 2PQN - PN  */
fmm_status_t fmm_plan_stats(const fmm_plan_t* plan, double out[8]);

/* out[0..7] as fmm_plan_stats, then the split by launch:
   [8]  flops of the leaf-level launch (the leaf products, fused or not)
   [9]  addition HBM bytes evaluated inside the fused leaf-level launch (0 if not fused)
   [10] number of fused leaf-level launches per execute (0 or 1)
   [11] addition bytes of the separate formation kernels (levels below the fused one)
   [12] addition bytes of the separate assembly kernels
   [13] flops of the peel-strip products
   [14] 1 if the last two levels are collapsed (collapse_levels), else 0
   [15] 1 if the last split's rows were peeled to 128-row-aligned leaves (peel_tiles, R7c) */
fmm_status_t fmm_plan_stats_ex(const fmm_plan_t* plan, double out[16]);

/* The same, extensible: fills out[0 .. min(n, 19) - 1]; out[0..15] as fmm_plan_stats_ex, then
   [16] 1 if the output step is fused into the leaf GEMM (fuse_output applied), else 0;
   [17] 1 if the last two levels' assembly runs as one pass (collapse_levels: with the formation for
        the <2,2,2> family, or alone -- the wide warp-per-column kernel, FMM_WIDE_ASM=1 -- for base
        cases with MN <= 16), else 0;
   [18] 1 if the plan runs the whole step as one launch (small_fused applied), else 0. */
fmm_status_t fmm_plan_stats_ex2(const fmm_plan_t* plan, double* out, int n);

/* Cost model (host only, no allocation): predicted milliseconds of a plan of `alg` for the problem
   on one B200 -- leaf DMMA GEMM tile schedule (wave quantisation, tile widths), streaming addition
   traffic at the measured HBM rate, peel strips, launch costs; the recursion stops where
   plan_create stops (*used_levels, may be NULL).  The paper's cutoff question (Sec. 3.4,
   P:741-759): compare levels = 0, 1, 2, ... */
fmm_status_t fmm_plan_predict(const fmm_alg* alg, int64_t P, int64_t Q, int64_t Nc, int levels, int layout, double* ms,
                              int* used_levels);

/* Shape matching: over the candidate algorithms, their six Prop. 1/2
   permutations and levels 1..max_levels, the predicted-fastest plan, or the classical GEMM
   (*alg_index = -1, *levels = 0) when nothing beats it.  *perm is for fmm_alg_permute. */
fmm_status_t fmm_select(const fmm_alg* const* algs, int nalgs, int64_t P, int64_t Q, int64_t Nc, int max_levels, int layout,
                        int* alg_index, int* perm, int* levels, double* ms);

/* Host-only check (no device work): generate and NVRTC-compile, for sm_100a, the fused
   leaf-level kernel of `alg` (fuse_leaf_level = 1) for the given layout, CSE setting and GEMM tile
   width (128, 112, 96, 80 or 64).  FMM_E_CUDA with the compiler log on failure. */
fmm_status_t fmm_fused_compile_check(const fmm_alg* alg, int layout, int cse, int bn);
/* The same for ring depth ks (16, 32 or 48) and fuse_leaf_level mode (1 = addition CTAs,
   2 = background jobs in the GEMM CTAs' spare warps).  fmm_fused_compile_check is (ks 16, mode 1). */
fmm_status_t fmm_fused_compile_check_ex(const fmm_alg* alg, int layout, int cse, int bn, int ks, int mode);

/* Execute C <- A*B (beta = 0: C is overwritten).  A, B, C are device pointers on the plan's
   device laid out per opt->layout; C must not alias A or B.  Leading dimensions in elements:
   row-major lda >= Q, ldb >= Nc, ldc >= Nc; column-major lda >= P, ldb >= Q, ldc >= P.
   `stream` is a cudaStream_t (NULL = legacy default stream).  Stream-ordered and
   asynchronous: returns after enqueueing; launch errors return FMM_E_CUDA, and asynchronous
   kernel faults surface at the next fmm_* call on that plan or at fmm_sync.
   With shard_count > 1 the result is this shard's partial product (sum over shards = A*B). */
fmm_status_t fmm_execute(fmm_plan_t* plan, const double* A, int64_t lda, const double* B, int64_t ldb,
                         double* C, int64_t ldc, void* stream);

/* Same, timing every launch with CUDA events on `stream` (plain launches, no CUDA graph; blocking:
   synchronises the stream) and summing the launch times by phase: ms[0] = formation kernels,
   ms[1] = leaf products (GEMM, or the fused leaf-level launch), ms[2] = assembly kernels,
   ms[3] = peel-strip GEMMs, ms[4] = total from the first launch to the end of the step, including a
   distributed plan's combine (whose exposed part is ms[4] - ms[0..3]). */
fmm_status_t fmm_execute_timed(fmm_plan_t* plan, const double* A, int64_t lda, const double* B,
                               int64_t ldb, double* C, int64_t ldc, void* stream, float ms[5]);

/* Diagnostics: fmm_execute with an event after every launch (plain launches, blocking); for the
   first min(*n, max) launches: kind[q] (0 A formation, 1 B formation, 2 leaf GEMM, 3 assembly,
   4 peel strips, 5 thin products on CUDA cores, 6 fused leaf level, 7 combine, 8 zeroing for
   fuse_output, 9 the one-launch small_fused step), level[q] (recursion level) and ms[q]; *n = the
   number of launches. */
fmm_status_t fmm_execute_profile(fmm_plan_t* plan, const double* A, int64_t lda, const double* B, int64_t ldb,
                                 double* C, int64_t ldc, void* stream, int max, int* kind, int* level, float* ms,
                                 int* n);

/* Same as fmm_execute, additionally recording four caller-created cudaEvent_t on `stream`
   (non-blocking): events[0] before the first kernel, [1] after the formation kernels, [2] after
   the leaf GEMM, [3] after the assembly and peel-strip kernels, before a distributed plan's
   combine completes (an event the caller records after the call closes the combine phase).
   Plain launches (no CUDA graph).  Used to time the phases without synchronising. */
fmm_status_t fmm_execute_events(fmm_plan_t* plan, const double* A, int64_t lda, const double* B,
                                int64_t ldb, double* C, int64_t ldc, void* stream, void* events[4]);

/* Host-memory execution (the end-to-end path): copies A and B (host memory) to device staging
   buffers owned by the plan, executes on `stream`, and copies C back to host; synchronises
   before returning. */
fmm_status_t fmm_execute_host(fmm_plan_t* plan, const double* A, int64_t lda, const double* B,
                              int64_t ldb, double* C, int64_t ldc, void* stream);

/* Pipelined host-memory execution: enqueue the H2D copies (plan-owned copy-in stream), the
   computation (`stream`) and the D2H copy (plan-owned copy-out stream) and return.  The plan
   alternates two staging sets, so back-to-back calls overlap copy-in of one problem, compute of
   another and copy-out of a third.  Host buffers must be pinned for overlap and must stay valid
   and unmodified (C unread) until fmm_sync(plan) returns. */
fmm_status_t fmm_execute_host_async(fmm_plan_t* plan, const double* A, int64_t lda, const double* B,
                                    int64_t ldb, double* C, int64_t ldc, void* stream);

/* Block until every fmm_execute on the plan has finished; reports asynchronous faults. */
fmm_status_t fmm_sync(fmm_plan_t* plan);
void fmm_plan_destroy(fmm_plan_t* plan);

/* Short spellings of the north-star API: fmm_plan(alg U/V/W, M,K,N, levels) and
   fmm_execute(A,B,C) (BASELINE.json).  fmm_plan == fmm_plan_create with default options on
   the current device; fmm_exec == fmm_execute with tight leading dimensions on the default
   stream. */
fmm_status_t fmm_plan(const fmm_alg* alg, int64_t M, int64_t K, int64_t N, int levels, fmm_plan_t** out);
fmm_status_t fmm_exec(fmm_plan_t* plan, const double* A, const double* B, double* C);

/* ---- leaf sharding arithmetic (host only, Sec. 4.3) --------------------------- */

/* For R^L leaves over G workers: *bfs = R^L - (R^L mod G) leaves split evenly (contiguous,
   r_1-major), *dfs = R^L mod G leaves split by rows over all G. */
fmm_status_t fmm_hybrid_split(int64_t R, int L, int64_t G, int64_t* bfs, int64_t* dfs);

/* The leaf share of worker g of G (the partition every sharded plan uses): for each of the
   `leaves` leaves (index r_1-major), rows [r0[z], r1[z]) of its product belong to worker g
   (r0 == r1: none).  The first leaves - (leaves mod G) leaves go whole to one worker each in
   contiguous equal ranges; each remaining leaf is split by rows over all G.  Host only. */
fmm_status_t fmm_shard_leaf_rows(int64_t leaves, int64_t rows, int64_t G, int64_t g, int64_t* r0, int64_t* r1);

/* ---- kernels usable on their own (device pointers, stream-ordered) ---------------------- */

/* Classical product C = alpha*A*B + beta*C with the library's DMMA GEMM kernel (row-major,
   mma.sync f64 on the FP64 tensor pipe).  The L = 0 path of a plan. */
fmm_status_t fmm_dgemm(int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda,
                       const double* B, int64_t ldb, double beta, double* C, int64_t ldc, void* stream);

/* Measure the FP64 ceilings of the current device with this library's microbenchmark kernels
   (independent mma.sync.m8n8k4.f64 chains; independent DFMA chains), ~50 ms.  The roofline
   denominator for the leaf GEMM (MEASURED_PEAKS.json carries no FP64 figure). */
fmm_status_t fmm_probe_fp64_peak(double* dmma_tflops, double* dfma_tflops);

const char* fmm_last_error(void);
const char* fmm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FMM_H */
