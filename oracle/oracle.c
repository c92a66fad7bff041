/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU evaluation of what the hot path computes, written from
 * the paper (arXiv 1409.2908, /root/reference/PAPER.md, cited as P:<line>).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load this.
 * It shares no code, header, table or helper with the CUDA path (paper_1409_2908_b200/).
 *
 * Arithmetic: IEEE-754 binary64, round-to-nearest-even, compiled with -ffp-contract=off so no
 * FMA contraction happens (reading R9).  Summation orders are fixed and stated per
 * function so results are reproducible bit for bit.
 *
 * Layout: every matrix argument is a (pointer, row stride, column stride) triple, so both
 * row-major (rs = ld, cs = 1) and column-major (rs = 1, cs = ld) storage are addressed through
 * the same logical (row, col) element A(i,j) = A[i*rs + j*cs].
 *
 * Functions
 *   oracle_classical   C = A*B by the definition C_ij = sum_q A_iq B_qj
 *   oracle_fast        recursive evaluation of a bilinear <M,K,N;R> algorithm (U,V,W) for L
 *                      steps, dynamic peeling at every level                     (P:295-331,
 *                      P:553-583)
 *   oracle_fast_entry  one entry C_ij of exactly the same evaluation, computed lazily (used to
 *                      sample full-size problems); bit-identical to oracle_fast by construction
 *   oracle_flops       the number of floating-point operations oracle_fast performs
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int M, K, N, R;
  const double* U; /* MK x R, row-major: U[i*R + r] = u_ir, i = a*K + b for A-block (a,b) */
  const double* V; /* KN x R: j = b*N + c for B-block (b,c) */
  const double* W; /* MN x R: k = a*N + c for C-block (a,c) */
} oalg;

/* ---------------------------------------------------------------------------------------- */
/* Classical product, the definition.  C_ij = sum_{q=0}^{Q-1} A_iq * B_qj, the sum  */
/* taken q ascending starting from 0.0.  Parallel over rows only, so the per-entry order is    */
/* fixed.                                                                                       */
/* ---------------------------------------------------------------------------------------- */
/* Small loops run on one thread: the threads only partition independent element positions, so
   this changes nothing in the arithmetic, but an oversubscribed host otherwise spends seconds per
   tiny parallel region waiting for descheduled threads. */
#define OMP_MIN_WORK (1 << 16)

void oracle_classical(int64_t P, int64_t Q, int64_t Nc,
                      const double* A, int64_t ars, int64_t acs,
                      const double* B, int64_t brs, int64_t bcs,
                      double* C, int64_t crs, int64_t ccs) {
#pragma omp parallel for schedule(dynamic, 1) if (P * Q * Nc >= OMP_MIN_WORK)
  for (int64_t i = 0; i < P; ++i) {
    double* acc = (double*)malloc(sizeof(double) * (Nc > 0 ? Nc : 1));
    for (int64_t j = 0; j < Nc; ++j) acc[j] = 0.0;
    for (int64_t q = 0; q < Q; ++q) {
      const double a = A[i * ars + q * acs];
      const double* brow = B + q * brs;
      for (int64_t j = 0; j < Nc; ++j) acc[j] = acc[j] + a * brow[j * bcs];
    }
    for (int64_t j = 0; j < Nc; ++j) C[i * crs + j * ccs] = acc[j];
    free(acc);
  }
}

/* One step of an addition chain: the first nonzero coefficient initialises the  */
/* result (copy / negate / scale), later ones add, subtract, or add a scaled term.           */
static inline double chain_first(double c, double x) {
  if (c == 1.0) return x;
  if (c == -1.0) return -x;
  return c * x;
}
static inline double chain_next(double acc, double c, double x) {
  if (c == 1.0) return acc + x;
  if (c == -1.0) return acc - x;
  return acc + c * x;
}

/* ---------------------------------------------------------------------------------------- */
/* Recursive fast multiplication, L steps, dynamic peeling at every level.        */
/*  1. If L == 0 or a dimension is smaller than the base case: classical (R10/R18). */
/*  2. Core P' = M*floor(P/M), Q' = K*floor(Q/K), N' = N*floor(N/N); blocks p x q, q x n.      */
/*  3. For r = 1..R (ascending): S_r = sum_i u_ir A_i, T_r = sum_j v_jr B_j (i, j ascending,  */
/*     first term initialises), M_r = fast(S_r, T_r, L-1).  No CSE, no scalar piping.        */
/*  4. C_k = sum_r w_kr M_r (r ascending, first term initialises).                            */
/*  5. Peeling fix-ups, all classical (SPEC S:287-295 reading, R7):                 */
/*     (a) Q' < Q: C[0:P',0:N'] = C[0:P',0:N'] + A[0:P',Q':Q] * B[Q':Q,0:N']                   */
/*     (b) P' < P: C[P':P, :]   = A[P':P, :] * B                                               */
/*     (c) N' < N: C[0:P', N':N] = A[0:P', :] * B[:, N':N]                                     */
/* ---------------------------------------------------------------------------------------- */
static void fast_rec(const oalg* g, int L, int64_t P, int64_t Q, int64_t Nc,
                     const double* A, int64_t ars, int64_t acs,
                     const double* B, int64_t brs, int64_t bcs,
                     double* C, int64_t crs, int64_t ccs) {
  const int M = g->M, K = g->K, N = g->N, R = g->R;
  if (L == 0 || P < M || Q < K || Nc < N) {
    oracle_classical(P, Q, Nc, A, ars, acs, B, brs, bcs, C, crs, ccs);
    return;
  }
  const int64_t P1 = M * (P / M), Q1 = K * (Q / K), N1 = N * (Nc / N);
  const int64_t p = P1 / M, q = Q1 / K, n = N1 / N;
  double* S = (double*)malloc(sizeof(double) * p * q);
  double* T = (double*)malloc(sizeof(double) * q * n);
  double* Mr = (double*)malloc(sizeof(double) * (size_t)R * p * n);
  for (int r = 0; r < R; ++r) {
    int first = 1;
    for (int i = 0; i < M * K; ++i) {
      const double u = g->U[i * R + r];
      if (u == 0.0) continue;
      const double* blk = A + (i / K) * p * ars + (i % K) * q * acs;
#pragma omp parallel for if (p * q >= OMP_MIN_WORK)
      for (int64_t x = 0; x < p; ++x)
        for (int64_t y = 0; y < q; ++y) {
          const double v = blk[x * ars + y * acs];
          S[x * q + y] = first ? chain_first(u, v) : chain_next(S[x * q + y], u, v);
        }
      first = 0;
    }
    if (first) memset(S, 0, sizeof(double) * p * q); /* zero column: S_r = 0 */
    first = 1;
    for (int j = 0; j < K * N; ++j) {
      const double v = g->V[j * R + r];
      if (v == 0.0) continue;
      const double* blk = B + (j / N) * q * brs + (j % N) * n * bcs;
#pragma omp parallel for if (q * n >= OMP_MIN_WORK)
      for (int64_t x = 0; x < q; ++x)
        for (int64_t y = 0; y < n; ++y) {
          const double b = blk[x * brs + y * bcs];
          T[x * n + y] = first ? chain_first(v, b) : chain_next(T[x * n + y], v, b);
        }
      first = 0;
    }
    if (first) memset(T, 0, sizeof(double) * q * n);
    fast_rec(g, L - 1, p, q, n, S, q, 1, T, n, 1, Mr + (size_t)r * p * n, n, 1);
  }
  for (int k = 0; k < M * N; ++k) {
    double* cb = C + (k / N) * p * crs + (k % N) * n * ccs;
    int first = 1;
    for (int r = 0; r < R; ++r) {
      const double w = g->W[k * R + r];
      if (w == 0.0) continue;
      const double* mb = Mr + (size_t)r * p * n;
#pragma omp parallel for if (p * n >= OMP_MIN_WORK)
      for (int64_t x = 0; x < p; ++x)
        for (int64_t y = 0; y < n; ++y) {
          const double m = mb[x * n + y];
          double* c = cb + x * crs + y * ccs;
          *c = first ? chain_first(w, m) : chain_next(*c, w, m);
        }
      first = 0;
    }
    if (first)
      for (int64_t x = 0; x < p; ++x)
        for (int64_t y = 0; y < n; ++y) cb[x * crs + y * ccs] = 0.0;
  }
  free(S); free(T); free(Mr);
  if (Q1 < Q) { /* (a) rank-(Q-Q') update of the core */
    double* tmp = (double*)malloc(sizeof(double) * P1 * N1);
    oracle_classical(P1, Q - Q1, N1, A + Q1 * acs, ars, acs, B + Q1 * brs, brs, bcs, tmp, N1, 1);
    for (int64_t x = 0; x < P1; ++x)
      for (int64_t y = 0; y < N1; ++y) C[x * crs + y * ccs] = C[x * crs + y * ccs] + tmp[x * N1 + y];
    free(tmp);
  }
  if (P1 < P) /* (b) trailing rows */
    oracle_classical(P - P1, Q, Nc, A + P1 * ars, ars, acs, B, brs, bcs, C + P1 * crs, crs, ccs);
  if (N1 < Nc) /* (c) trailing columns of the first P' rows */
    oracle_classical(P1, Q, Nc - N1, A, ars, acs, B + N1 * bcs, brs, bcs, C + N1 * ccs, crs, ccs);
}

void oracle_fast(int64_t P, int64_t Q, int64_t Nc,
                 const double* A, int64_t ars, int64_t acs,
                 const double* B, int64_t brs, int64_t bcs,
                 double* C, int64_t crs, int64_t ccs,
                 int M, int K, int N, int R, const double* U, const double* V, const double* W, int L) {
  oalg g = {M, K, N, R, U, V, W};
  fast_rec(&g, L, P, Q, Nc, A, ars, acs, B, brs, bcs, C, crs, ccs);
}

/* ---------------------------------------------------------------------------------------- */
/* Lazy single-entry evaluation of exactly the computation of fast_rec.                       */
/* An operand at depth d is the virtual matrix S_{r_1..r_d}; its element (x, y) is the same    */
/* addition chain fast_rec applies, evaluated on the parent's elements (same order, same        */
/* first-term rule), so every intermediate is rounded identically.                             */
/* ---------------------------------------------------------------------------------------- */
#define OMAXL 8
typedef struct {
  const oalg* g;
  const double* A; int64_t ars, acs;
  const double* B; int64_t brs, bcs;
  int path[OMAXL + 1];      /* r at depths 1..d */
  int64_t ap[OMAXL + 1], aq[OMAXL + 1]; /* dims of the A-side operand at depth d (rows, cols) */
  int64_t bq[OMAXL + 1], bn[OMAXL + 1]; /* dims of the B-side operand at depth d */
} ectx;

static double elemA(const ectx* c, int d, int64_t x, int64_t y) {
  if (d == 0) return c->A[x * c->ars + y * c->acs];
  const oalg* g = c->g;
  const int r = c->path[d];
  const int64_t p = c->ap[d], q = c->aq[d];
  int first = 1;
  double s = 0.0;
  for (int i = 0; i < g->M * g->K; ++i) {
    const double u = g->U[i * g->R + r];
    if (u == 0.0) continue;
    const double v = elemA(c, d - 1, (i / g->K) * p + x, (i % g->K) * q + y);
    s = first ? chain_first(u, v) : chain_next(s, u, v);
    first = 0;
  }
  return s; /* a zero column gives 0.0, as the memset in fast_rec */
}

static double elemB(const ectx* c, int d, int64_t x, int64_t y) {
  if (d == 0) return c->B[x * c->brs + y * c->bcs];
  const oalg* g = c->g;
  const int r = c->path[d];
  const int64_t q = c->bq[d], n = c->bn[d];
  int first = 1;
  double s = 0.0;
  for (int j = 0; j < g->K * g->N; ++j) {
    const double v = g->V[j * g->R + r];
    if (v == 0.0) continue;
    const double b = elemB(c, d - 1, (j / g->N) * q + x, (j % g->N) * n + y);
    s = first ? chain_first(v, b) : chain_next(s, v, b);
    first = 0;
  }
  return s;
}

/* classical dot product over q in [q0, q1), ascending from 0.0, as oracle_classical does */
static double dotAB(const ectx* c, int d, int64_t x, int64_t y, int64_t q0, int64_t q1) {
  double acc = 0.0;
  for (int64_t q = q0; q < q1; ++q) acc = acc + elemA(c, d, x, q) * elemB(c, d, q, y);
  return acc;
}

static double entry_rec(ectx* c, int d, int Lleft, int64_t P, int64_t Q, int64_t Nc, int64_t x, int64_t y) {
  const oalg* g = c->g;
  const int M = g->M, K = g->K, N = g->N, R = g->R;
  if (Lleft == 0 || P < M || Q < K || Nc < N) return dotAB(c, d, x, y, 0, Q);
  const int64_t P1 = M * (P / M), Q1 = K * (Q / K), N1 = N * (Nc / N);
  const int64_t p = P1 / M, q = Q1 / K, n = N1 / N;
  if (x >= P1 || y >= N1) return dotAB(c, d, x, y, 0, Q); /* strips (b), (c) */
  const int a = (int)(x / p), cc = (int)(y / n);
  const int k = a * N + cc;
  c->ap[d + 1] = p; c->aq[d + 1] = q; c->bq[d + 1] = q; c->bn[d + 1] = n;
  int first = 1;
  double val = 0.0;
  for (int r = 0; r < R; ++r) {
    const double w = g->W[k * R + r];
    if (w == 0.0) continue;
    c->path[d + 1] = r;
    const double m = entry_rec(c, d + 1, Lleft - 1, p, q, n, x - a * p, y - cc * n);
    val = first ? chain_first(w, m) : chain_next(val, w, m);
    first = 0;
  }
  if (Q1 < Q) val = val + dotAB(c, d, x, y, Q1, Q); /* fix-up (a) */
  return val;
}

void oracle_fast_entries(int64_t P, int64_t Q, int64_t Nc,
                         const double* A, int64_t ars, int64_t acs,
                         const double* B, int64_t brs, int64_t bcs,
                         int M, int K, int N, int R, const double* U, const double* V, const double* W, int L,
                         int64_t count, const int64_t* rows, const int64_t* cols, double* out) {
  oalg g = {M, K, N, R, U, V, W};
#pragma omp parallel for schedule(dynamic, 1) if (count >= 64)
  for (int64_t e = 0; e < count; ++e) {
    ectx c;
    memset(&c, 0, sizeof(c));
    c.g = &g; c.A = A; c.ars = ars; c.acs = acs; c.B = B; c.brs = brs; c.bcs = bcs;
    out[e] = entry_rec(&c, 0, L < OMAXL ? L : OMAXL, P, Q, Nc, rows[e], cols[e]);
  }
}

/* ---------------------------------------------------------------------------------------- */
/* Flop count of oracle_fast.  Classical P x Q x N: P*N*(2Q-1) (one multiply per   */
/* term, Q-1 additions).  An addition chain with k nonzero coefficients costs k-1 additions    */
/* per element; non-unit coefficients cost one multiply per element (inactive multiplies;     */
/* none for +-1).  Peeling fix-up (a) adds P'N' additions for the update.               */
/* ---------------------------------------------------------------------------------------- */
static double classical_flops(int64_t P, int64_t Q, int64_t Nc) {
  if (P <= 0 || Nc <= 0 || Q <= 0) return 0.0;
  return (double)P * (double)Nc * (2.0 * (double)Q - 1.0);
}

static double chain_flops(const double* X, int rows, int R, int r, double elems) {
  int nz = 0, scaled = 0;
  for (int i = 0; i < rows; ++i) {
    const double c = X[i * R + r];
    if (c == 0.0) continue;
    ++nz;
    if (c != 1.0 && c != -1.0) ++scaled;
  }
  return (nz > 0 ? (double)(nz - 1) : 0.0) * elems + (double)scaled * elems;
}

static double flops_rec(const oalg* g, int L, int64_t P, int64_t Q, int64_t Nc) {
  const int M = g->M, K = g->K, N = g->N, R = g->R;
  if (L == 0 || P < M || Q < K || Nc < N) return classical_flops(P, Q, Nc);
  const int64_t P1 = M * (P / M), Q1 = K * (Q / K), N1 = N * (Nc / N);
  const int64_t p = P1 / M, q = Q1 / K, n = N1 / N;
  double f = 0.0;
  for (int r = 0; r < R; ++r) {
    f += chain_flops(g->U, M * K, R, r, (double)p * q);
    f += chain_flops(g->V, K * N, R, r, (double)q * n);
    f += flops_rec(g, L - 1, p, q, n);
  }
  for (int k = 0; k < M * N; ++k) {
    int nz = 0, scaled = 0;
    for (int r = 0; r < R; ++r) {
      const double w = g->W[k * R + r];
      if (w == 0.0) continue;
      ++nz;
      if (w != 1.0 && w != -1.0) ++scaled;
    }
    f += (double)((nz > 0 ? nz - 1 : 0) + scaled) * (double)p * n;
  }
  if (Q1 < Q) f += classical_flops(P1, Q - Q1, N1) + (double)P1 * N1;
  if (P1 < P) f += classical_flops(P - P1, Q, Nc);
  if (N1 < Nc) f += classical_flops(P1, Q, Nc - N1);
  return f;
}

double oracle_flops(int64_t P, int64_t Q, int64_t Nc, int M, int K, int N, int R,
                    const double* U, const double* V, const double* W, int L) {
  oalg g = {M, K, N, R, U, V, W};
  return flops_rec(&g, L, P, Q, Nc);
}
