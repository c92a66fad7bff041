// L1: algorithm objects — exact rational coefficients, exact Brent validation, the Prop. 1
// transpose used for column-major problems, and the S:190 text format.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>

#include "fmm_internal.h"

namespace fmm {

static __int128 gcd128(__int128 a, __int128 b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b) {
    __int128 t = a % b;
    a = b;
    b = t;
  }
  return a;
}
// Every numerator and denominator stays within +-2^100; each product or sum below is computed with
// the overflow-checked builtins, so an algorithm whose coefficients outgrow 128 bits is refused
// (FMM_E_UNSUPPORTED) instead of being misjudged by a wrapped intermediate.
static const __int128 kLimit = (__int128)1 << 100;
static void check_range(__int128 v) {
  if (v > kLimit || v < -kLimit) throw Error(FMM_E_UNSUPPORTED, "rational coefficient arithmetic overflow");
}
static __int128 mul_checked(__int128 a, __int128 b) {
  __int128 r;
  if (__builtin_mul_overflow(a, b, &r)) throw Error(FMM_E_UNSUPPORTED, "rational coefficient arithmetic overflow");
  return r;
}
static __int128 add_checked(__int128 a, __int128 b) {
  __int128 r;
  if (__builtin_add_overflow(a, b, &r)) throw Error(FMM_E_UNSUPPORTED, "rational coefficient arithmetic overflow");
  return r;
}

Rat rat_make(__int128 n, __int128 d) {
  if (d == 0) throw Error(FMM_E_INVALID_ARG, "zero denominator");
  if (d < 0) n = -n, d = -d;
  __int128 g = gcd128(n, d);
  if (g > 1) n /= g, d /= g;
  if (n == 0) d = 1;
  check_range(n);
  check_range(d);
  return Rat{n, d};
}
Rat rat_add(Rat a, Rat b) {
  if (a.n == 0) return b;
  if (b.n == 0) return a;
  __int128 g = gcd128(a.d, b.d);
  return rat_make(add_checked(mul_checked(a.n, b.d / g), mul_checked(b.n, a.d / g)), mul_checked(a.d / g, b.d));
}
Rat rat_mul(Rat a, Rat b) {
  if (a.n == 0 || b.n == 0) return Rat{0, 1};
  __int128 g1 = gcd128(a.n, b.d), g2 = gcd128(b.n, a.d);
  return rat_make(mul_checked(a.n / g1, b.n / g2), mul_checked(a.d / g2, b.d / g1));
}

// T_ijk of the <M,K,N> matmul tensor from the index conditions of P:415-421 (0-based).
static inline int tensor_entry(int M, int K, int N, int i, int j, int k) {
  (void)M;
  return (i % K == j / N) && (j % N == k % N) && (i / K == k / N);
}

void alg_validate_exact(const fmm_alg& a) {
  const int M = a.M, K = a.K, N = a.N, R = a.R;
  long long bad = 0;
  std::string first;
  std::vector<Rat> uv(R);
  for (int i = 0; i < M * K; ++i)
    for (int j = 0; j < K * N; ++j) {
      for (int r = 0; r < R; ++r) uv[r] = rat_mul(a.U[i * R + r], a.V[j * R + r]);
      for (int k = 0; k < M * N; ++k) {
        Rat s{0, 1};
        for (int r = 0; r < R; ++r)
          if (uv[r].n != 0 && a.W[k * R + r].n != 0) s = rat_add(s, rat_mul(uv[r], a.W[k * R + r]));
        const int t = tensor_entry(M, K, N, i, j, k);
        if (!(s.d == 1 && s.n == t)) {
          if (bad == 0)
            first = "(i,j,k)=(" + std::to_string(i) + "," + std::to_string(j) + "," + std::to_string(k) + ")";
          ++bad;
        }
      }
    }
  if (bad)
    throw Error(FMM_E_NOT_EXACT, "algorithm violates " + std::to_string(bad) +
                                     " Brent equations (P:313-319); first at " + first);
}

static void fill_doubles(fmm_alg& a) {
  auto conv = [](const std::vector<Rat>& X, std::vector<double>& Y) {
    Y.resize(X.size());
    for (size_t i = 0; i < X.size(); ++i) Y[i] = rat_to_double(X[i]);
  };
  conv(a.U, a.Ud);
  conv(a.V, a.Vd);
  conv(a.W, a.Wd);
}

// P_{IxJ} X: row (c*I + a) of the result is row (a*J + c) of X.
static std::vector<Rat> perm_rows(const std::vector<Rat>& X, int I, int J, int R) {
  std::vector<Rat> out(X.size());
  for (int a = 0; a < I; ++a)
    for (int c = 0; c < J; ++c)
      for (int r = 0; r < R; ++r) out[(c * I + a) * R + r] = X[(a * J + c) * R + r];
  return out;
}

fmm_alg* alg_transpose_prop1(const fmm_alg& a) {
  // Prop. 1: <P_{KxN} V, P_{MxK} U, P_{MxN} W> is an algorithm for <N,K,M>.
  auto* t = new fmm_alg;
  t->M = a.N;
  t->K = a.K;
  t->N = a.M;
  t->R = a.R;
  t->U = perm_rows(a.V, a.K, a.N, a.R);
  t->V = perm_rows(a.U, a.M, a.K, a.R);
  t->W = perm_rows(a.W, a.M, a.N, a.R);
  fill_doubles(*t);
  return t;
}

fmm_alg* alg_cycle_prop2(const fmm_alg& a) {
  // Prop. 2: <P_{MxN} W, U, P_{KxN} V> is an algorithm for <N,M,K>.
  auto* t = new fmm_alg;
  t->M = a.N;
  t->K = a.M;
  t->N = a.K;
  t->R = a.R;
  t->U = perm_rows(a.W, a.M, a.N, a.R);
  t->V = a.U;
  t->W = perm_rows(a.V, a.K, a.N, a.R);
  fill_doubles(*t);
  return t;
}

static fmm_alg* alg_from_rats(int M, int K, int N, int R, std::vector<Rat> U, std::vector<Rat> V,
                              std::vector<Rat> W) {
  if (M < 1 || K < 1 || N < 1 || M > 16 || K > 16 || N > 16 || R < 1 || R > 4096)
    throw Error(FMM_E_INVALID_ARG, "algorithm dims out of range (1<=M,K,N<=16, 1<=R<=4096)");
  std::unique_ptr<fmm_alg> a(new fmm_alg);
  a->M = M;
  a->K = K;
  a->N = N;
  a->R = R;
  a->U = std::move(U);
  a->V = std::move(V);
  a->W = std::move(W);
  alg_validate_exact(*a);
  fill_doubles(*a);
  return a.release();
}

static Rat parse_rational(const std::string& tok, int line) {
  const char* s = tok.c_str();
  char* end = nullptr;
  long long n = strtoll(s, &end, 10);
  long long d = 1;
  if (end == s) throw Error(FMM_E_PARSE, "line " + std::to_string(line) + ": bad coefficient '" + tok + "'");
  if (*end == '/') {
    const char* s2 = end + 1;
    d = strtoll(s2, &end, 10);
    if (end == s2 || d <= 0)
      throw Error(FMM_E_PARSE, "line " + std::to_string(line) + ": bad denominator in '" + tok + "'");
  }
  if (*end != '\0') {
    if (strchr(tok.c_str(), 'L'))
      throw Error(FMM_E_UNSUPPORTED, "line " + std::to_string(line) + ": APA (lambda) coefficients unsupported");
    throw Error(FMM_E_PARSE, "line " + std::to_string(line) + ": bad coefficient '" + tok + "'");
  }
  return rat_make(n, d);
}

static fmm_alg* alg_parse_file(const char* path) {
  std::ifstream f(path);
  if (!f) throw Error(FMM_E_INVALID_ARG, std::string("cannot open ") + path);
  std::string ln;
  int line = 0;
  int hdr[4] = {0, 0, 0, 0};
  bool have_hdr = false;
  std::vector<std::vector<Rat>> rows;
  while (std::getline(f, ln)) {
    ++line;
    auto h = ln.find('#');
    if (h != std::string::npos) ln = ln.substr(0, h);
    std::istringstream ss(ln);
    std::vector<std::string> toks;
    std::string t;
    while (ss >> t) toks.push_back(t);
    if (toks.empty()) continue;
    if (!have_hdr) {
      if (toks.size() < 4) throw Error(FMM_E_PARSE, "line " + std::to_string(line) + ": header needs 'M K N R'");
      for (int q = 0; q < 4; ++q) {
        char* e = nullptr;
        hdr[q] = (int)strtol(toks[q].c_str(), &e, 10);
        if (*e) throw Error(FMM_E_PARSE, "line " + std::to_string(line) + ": bad header field '" + toks[q] + "'");
      }
      if (toks.size() > 4 && toks[4] == "apa") throw Error(FMM_E_UNSUPPORTED, "APA algorithms are not supported");
      if (toks.size() > 4 && toks[4] != "exact")
        throw Error(FMM_E_PARSE, "line " + std::to_string(line) + ": expected 'exact' or 'apa'");
      have_hdr = true;
      continue;
    }
    if ((int)toks.size() != hdr[3])
      throw Error(FMM_E_PARSE, "line " + std::to_string(line) + ": expected " + std::to_string(hdr[3]) +
                                   " entries, got " + std::to_string(toks.size()));
    std::vector<Rat> row;
    for (auto& tk : toks) row.push_back(parse_rational(tk, line));
    rows.push_back(std::move(row));
  }
  if (!have_hdr) throw Error(FMM_E_PARSE, "no header line");
  const int M = hdr[0], K = hdr[1], N = hdr[2], R = hdr[3];
  if (M < 1 || K < 1 || N < 1 || R < 1) throw Error(FMM_E_PARSE, "header dims must be positive");
  if ((int)rows.size() != M * K + K * N + M * N)
    throw Error(FMM_E_PARSE, "expected " + std::to_string(M * K + K * N + M * N) + " coefficient rows, got " +
                                 std::to_string(rows.size()));
  std::vector<Rat> U, V, W;
  for (int i = 0; i < (int)rows.size(); ++i) {
    auto& dst = i < M * K ? U : (i < M * K + K * N ? V : W);
    dst.insert(dst.end(), rows[i].begin(), rows[i].end());
  }
  return alg_from_rats(M, K, N, R, std::move(U), std::move(V), std::move(W));
}

thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }

}  // namespace fmm

using namespace fmm;

extern "C" {

const char* fmm_last_error(void) { return fmm::g_last_error.c_str(); }
const char* fmm_version(void) { return "fmm-b200 0.1 (sm_100a)"; }

fmm_status_t fmm_alg_create(int M, int K, int N, int R, const int64_t* U_num, const int64_t* U_den,
                            const int64_t* V_num, const int64_t* V_den, const int64_t* W_num,
                            const int64_t* W_den, fmm_alg** out) {
  FMM_API_BEGIN
  if (!out || !U_num || !V_num || !W_num) throw Error(FMM_E_INVALID_ARG, "null argument");
  *out = nullptr;
  if (M < 1 || K < 1 || N < 1 || R < 1 || M > 16 || K > 16 || N > 16 || R > 4096)
    throw Error(FMM_E_INVALID_ARG, "algorithm dims out of range");
  auto conv = [&](const int64_t* num, const int64_t* den, int rows) {
    std::vector<Rat> X((size_t)rows * R);
    for (size_t i = 0; i < X.size(); ++i) {
      const int64_t d = den ? den[i] : 1;
      if (d <= 0) throw Error(FMM_E_INVALID_ARG, "denominators must be positive");
      X[i] = rat_make(num[i], d);
    }
    return X;
  };
  *out = alg_from_rats(M, K, N, R, conv(U_num, U_den, M * K), conv(V_num, V_den, K * N), conv(W_num, W_den, M * N));
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_alg_load(const char* path, fmm_alg** out) {
  FMM_API_BEGIN
  if (!path || !out) throw Error(FMM_E_INVALID_ARG, "null argument");
  *out = nullptr;
  *out = alg_parse_file(path);
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_alg_permute(const fmm_alg* a, int perm, fmm_alg** out) {
  FMM_API_BEGIN
  if (!a || !out) throw Error(FMM_E_INVALID_ARG, "null argument");
  if (perm < 0 || perm > 5) throw Error(FMM_E_INVALID_ARG, "perm must be in [0, 5]");
  *out = nullptr;
  // 0 <M,K,N>, 1 P1 <N,K,M>, 2 P2 <N,M,K>, 3 P2 P2 <K,N,M>, 4 P1 P2 <K,M,N>, 5 P1 P2 P2 <M,N,K>
  std::unique_ptr<fmm_alg> t(new fmm_alg(*a));
  const int cycles = perm == 2 || perm == 4 ? 1 : perm == 3 || perm == 5 ? 2 : 0;
  for (int c = 0; c < cycles; ++c) t.reset(alg_cycle_prop2(*t));
  if (perm == 1 || perm == 4 || perm == 5) t.reset(alg_transpose_prop1(*t));
  alg_validate_exact(*t);  // the propositions are exact; re-checked anyway
  *out = t.release();
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_alg_info(const fmm_alg* a, int dims[4], int nnz[3]) {
  FMM_API_BEGIN
  if (!a) throw Error(FMM_E_INVALID_ARG, "null algorithm");
  if (dims) {
    dims[0] = a->M;
    dims[1] = a->K;
    dims[2] = a->N;
    dims[3] = a->R;
  }
  if (nnz) {
    auto c = [](const std::vector<Rat>& X) {
      int n = 0;
      for (auto& v : X) n += v.n != 0;
      return n;
    };
    nnz[0] = c(a->U);
    nnz[1] = c(a->V);
    nnz[2] = c(a->W);
  }
  return FMM_OK;
  FMM_API_END
}

void fmm_alg_destroy(fmm_alg* a) { delete a; }

fmm_status_t fmm_hybrid_split(int64_t R, int L, int64_t G, int64_t* bfs, int64_t* dfs) {
  FMM_API_BEGIN
  if (R < 1 || L < 0 || G < 1 || !bfs || !dfs) throw Error(FMM_E_INVALID_ARG, "bad hybrid split arguments");
  int64_t leaves = 1;
  for (int l = 0; l < L; ++l) {
    if (leaves > ((int64_t)1 << 50) / R) throw Error(FMM_E_UNSUPPORTED, "too many leaves");
    leaves *= R;
  }
  *dfs = leaves % G;       // BFS on the first R^L - (R^L mod P) leaves,
  *bfs = leaves - *dfs;    // DFS (all workers) on the remaining R^L mod P
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_shard_leaf_rows(int64_t leaves, int64_t rows, int64_t G, int64_t g, int64_t* r0, int64_t* r1) {
  FMM_API_BEGIN
  if (leaves < 1 || rows < 0 || G < 1 || g < 0 || g >= G || !r0 || !r1)
    throw Error(FMM_E_INVALID_ARG, "bad shard arguments");
  // HYBRID arithmetic with GPUs as the workers: the first leaves - (leaves mod G)
  // leaves are dealt out in contiguous, equal ranges (BFS part); each of the remaining
  // leaves mod G leaves is split by rows over all G workers (DFS part).
  const int64_t dfs = leaves % G, bfs = leaves - dfs, per = bfs / G;
  for (int64_t z = 0; z < leaves; ++z) {
    if (z < bfs) {
      const bool mine = z >= g * per && z < (g + 1) * per;
      r0[z] = 0;
      r1[z] = mine ? rows : 0;
    } else {
      r0[z] = rows * g / G;
      r1[z] = rows * (g + 1) / G;
    }
  }
  return FMM_OK;
  FMM_API_END
}

}  // extern "C"
