// flipsearch: offline search for exact bilinear matrix multiplication algorithms <M,K,N;R> with
// coefficients in {-1, 0, 1}, by a random walk on the flip graph of matmul tensor decompositions
// (the SURVEY's C2-tool; the paper's own search is ALS, which needs "hands-on tinkering"
// to reach discrete solutions -- the flip walk stays exact by construction).
//
// A scheme is a list of rank-one terms a (x) b (x) c, a in Z^{MK} (A-block weights, row i = a*K+b),
// b in Z^{KN} (B-block, j = b*N+c), c in Z^{MN} (C-block, k = a*N+c): the paper's row-major block
// vectorisation and Brent equations.  Moves (all identities on the tensor):
//   flip    a(x)b(x)c + a(x)b'(x)c'  ->  a(x)(b+b')(x)c + a(x)b'(x)(c'-c)   (any of the 3 factor slots)
//   reduce  a(x)b(x)c + a(x)b(x)c'   ->  a(x)b(x)(c+c')                     (rank - 1)
//   plus    a(x)b(x)c + a'(x)b'(x)c' ->  (a-a')(x)b(x)c + a'(x)b(x)c + a'(x)b'(x)c'  (rank + 1, to
//           escape a plateau)
// Entries must stay in {-1, 0, 1}; terms with a zero factor are dropped.  Starts from the classical
// rank-MKN scheme (or --from FILE), stops at --target, re-verifies the Brent equations in exact
// integer arithmetic and writes the S:190 text format.  tests/test_oracle_algebra.py re-checks every
// file in algs/ independently with fractions.Fraction.
//
//   g++ -O2 -std=c++17 -o tools/flipsearch tools/flipsearch.cpp
//   tools/flipsearch M K N TARGET [--seed S] [--plateau P] [--seconds T] [--out FILE] [--from FILE] [--best FILE]
// (about 3.5 M flips/s on one core at R ~ 40; a plateau of 5e6 flips finds <2,3,4;20> in seconds to minutes)
#include <algorithm>
#include <array>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

namespace {

constexpr int MAXD = 64;  // MK, KN, MN <= 64

// a {-1,0,1} vector as two bit masks
struct Vec {
  uint64_t p = 0, n = 0;
  bool zero() const { return (p | n) == 0; }
  Vec neg() const { return Vec{n, p}; }
  bool operator==(const Vec& o) const { return p == o.p && n == o.n; }
};
// x + s*y with s = +-1, if every entry stays in {-1,0,1}
bool add(const Vec& x, const Vec& y, int s, Vec* out) {
  const Vec ys = s > 0 ? y : y.neg();
  if ((x.p & ys.p) | (x.n & ys.n)) return false;  // 1+1 or -1-1
  const uint64_t cancel = (x.p & ys.n) | (x.n & ys.p);
  out->p = (x.p | ys.p) & ~cancel;
  out->n = (x.n | ys.n) & ~cancel;
  return true;
}
// +1 if x == y, -1 if x == -y, 0 otherwise
int same(const Vec& x, const Vec& y) {
  if (x == y) return 1;
  if (x == y.neg()) return -1;
  return 0;
}

struct Term {
  Vec f[3];  // a, b, c
};

struct Problem {
  int M, K, N;
  int dim(int s) const { return s == 0 ? M * K : s == 1 ? K * N : M * N; }
};

std::vector<Term> classical(const Problem& pr) {
  std::vector<Term> t;
  for (int a = 0; a < pr.M; ++a)
    for (int b = 0; b < pr.K; ++b)
      for (int c = 0; c < pr.N; ++c) {
        Term x;
        x.f[0].p = 1ull << (a * pr.K + b);
        x.f[1].p = 1ull << (b * pr.N + c);
        x.f[2].p = 1ull << (a * pr.N + c);
        t.push_back(x);
      }
  return t;
}

int entry(const Vec& v, int i) { return (v.p >> i & 1) ? 1 : (v.n >> i & 1) ? -1 : 0; }

// exact check of sum_r a_r (x) b_r (x) c_r == T (P:415-421 conditions, 0-based)
bool verify(const Problem& pr, const std::vector<Term>& t) {
  const int MK = pr.dim(0), KN = pr.dim(1), MN = pr.dim(2);
  for (int i = 0; i < MK; ++i)
    for (int j = 0; j < KN; ++j)
      for (int k = 0; k < MN; ++k) {
        long long s = 0;
        for (const auto& x : t) s += (long long)entry(x.f[0], i) * entry(x.f[1], j) * entry(x.f[2], k);
        const int a = i / pr.K, b = i % pr.K, b2 = j / pr.N, c = j % pr.N, a2 = k / pr.N, c2 = k % pr.N;
        const long long want = (b == b2 && a == a2 && c == c2) ? 1 : 0;
        if (s != want) return false;
      }
  return true;
}

struct Walker {
  Problem pr;
  std::vector<Term> t;
  std::mt19937_64 rng;

  // merge term r with any other term sharing two factors (up to sign); true if the rank dropped
  bool try_reduce(size_t r) {
    for (size_t s = 0; s < t.size(); ++s) {
      if (s == r) continue;
      for (int free = 0; free < 3; ++free) {
        const int u = (free + 1) % 3, v = (free + 2) % 3;
        const int su = same(t[r].f[u], t[s].f[u]), sv = same(t[r].f[v], t[s].f[v]);
        if (!su || !sv) continue;
        Vec m;
        if (!add(t[r].f[free], t[s].f[free], su * sv, &m)) continue;
        t[r].f[free] = m;
        t.erase(t.begin() + s);
        if (s < r) --r;
        if (t[r].f[free].zero()) t.erase(t.begin() + r);
        return true;
      }
    }
    return false;
  }

  // one random flip; returns true if it changed the scheme.  *ch0 / *ch1 are the indices of the two
  // modified terms afterwards (-1 where a term vanished), the only ones a reduction can now involve
  bool flip(long* ch0, long* ch1) {
    *ch0 = *ch1 = -1;
    const size_t R = t.size();
    const size_t r = rng() % R;
    const int slot = (int)(rng() % 3);
    // candidates sharing slot factor with r
    size_t cand[256];
    int nc = 0;
    for (size_t s = 0; s < R && nc < 256; ++s)
      if (s != r && same(t[r].f[slot], t[s].f[slot])) cand[nc++] = s;
    if (!nc) return false;
    const size_t s = cand[rng() % nc];
    const int sg = same(t[r].f[slot], t[s].f[slot]);
    // write t[s] with the same slot factor as t[r]: move the sign into the next slot
    const int u = (slot + 1) % 3, v = (slot + 2) % 3;
    Vec su = sg > 0 ? t[s].f[u] : t[s].f[u].neg();
    Vec sv = t[s].f[v];
    // a(x)b(x)c + a(x)b'(x)c'  ->  a(x)(b+b')(x)c + a(x)b'(x)(c'-c)   (u = b slot, v = c slot), or with u / v swapped
    const bool swap = rng() & 1;
    const int U = swap ? v : u, V = swap ? u : v;
    Vec b = t[r].f[U], c = t[r].f[V];
    Vec b2 = swap ? sv : su, c2 = swap ? su : sv;
    Vec nb, nc2;
    if (!add(b, b2, 1, &nb) || !add(c2, c, -1, &nc2)) return false;
    t[r].f[U] = nb;
    // t[s] = a (x) b' (x) (c' - c), expressed in t[s]'s own slots
    Term ns;
    ns.f[slot] = t[r].f[slot];
    ns.f[U] = b2;
    ns.f[V] = nc2;
    t[s] = ns;
    // drop zero terms (larger index first)
    const size_t hi = std::max(r, s), lo = std::min(r, s);
    auto dead = [&](size_t q) { return t[q].f[0].zero() || t[q].f[1].zero() || t[q].f[2].zero(); };
    const bool dhi = dead(hi), dlo = dead(lo);
    if (dhi) t.erase(t.begin() + hi);
    if (dlo) t.erase(t.begin() + lo);
    if (!dlo) *ch0 = (long)lo;
    if (!dhi) *ch1 = (long)hi - (dlo ? 1 : 0);
    return true;
  }

  bool plus() {
    const size_t R = t.size();
    const size_t r = rng() % R, s = rng() % R;
    if (r == s) return false;
    const int slot = (int)(rng() % 3);
    Vec d;
    if (!add(t[r].f[slot], t[s].f[slot], -1, &d) || d.zero()) return false;
    // x(x)y(x)z + x'(x)y'(x)z' -> (x - x')(x)y(x)z + x'(x)y(x)z + x'(x)y'(x)z'
    Term extra = t[r];
    extra.f[slot] = t[s].f[slot];
    t[r].f[slot] = d;
    t.push_back(extra);
    return true;
  }
};

// a scheme in the S:190 text format (comments after '#'; header "M K N R ..."; MK rows of U, KN rows of
// V, MN rows of W, R entries each, all in {-1, 0, 1}), e.g. a direct sum to start from
std::vector<Term> read_file(const char* path, const Problem& pr) {
  FILE* f = fopen(path, "r");
  if (!f) {
    perror(path);
    exit(2);
  }
  std::vector<std::vector<int>> rows;
  std::vector<int> header;
  char line[1 << 14];
  while (fgets(line, sizeof line, f)) {
    if (char* h = strchr(line, '#')) *h = 0;
    std::vector<int> v;
    for (char* tok = strtok(line, " \t\r\n"); tok; tok = strtok(nullptr, " \t\r\n")) {
      char* end = nullptr;
      const long x = strtol(tok, &end, 10);
      if (end && *end == 0) v.push_back((int)x);
    }
    if (v.empty()) continue;
    if (header.empty()) header = v;
    else rows.push_back(v);
  }
  fclose(f);
  if (header.size() < 4 || header[0] != pr.M || header[1] != pr.K || header[2] != pr.N) {
    fprintf(stderr, "%s: not a <%d,%d,%d> scheme\n", path, pr.M, pr.K, pr.N);
    exit(2);
  }
  const int R = header[3];
  if ((int)rows.size() != pr.dim(0) + pr.dim(1) + pr.dim(2)) {
    fprintf(stderr, "%s: expected %d coefficient rows\n", path, pr.dim(0) + pr.dim(1) + pr.dim(2));
    exit(2);
  }
  std::vector<Term> t(R);
  int row = 0;
  for (int s = 0; s < 3; ++s)
    for (int i = 0; i < pr.dim(s); ++i, ++row) {
      if ((int)rows[row].size() != R) {
        fprintf(stderr, "%s: row %d has %zu entries, want %d\n", path, row, rows[row].size(), R);
        exit(2);
      }
      for (int r = 0; r < R; ++r) {
        const int x = rows[row][r];
        if (x < -1 || x > 1) {
          fprintf(stderr, "%s: entry %d outside {-1, 0, 1}\n", path, x);
          exit(2);
        }
        if (x == 1) t[r].f[s].p |= 1ull << i;
        if (x == -1) t[r].f[s].n |= 1ull << i;
      }
    }
  return t;
}

void write_file(const char* path, const Problem& pr, const std::vector<Term>& t, unsigned long long seed,
                const char* from_desc) {
  FILE* f = fopen(path, "w");
  if (!f) {
    perror(path);
    exit(1);
  }
  fprintf(f, "# <%d,%d,%d;%zu> exact bilinear algorithm, entries in {-1,0,1}.\n", pr.M, pr.K, pr.N, t.size());
  fprintf(f, "# Found by tools/flipsearch.cpp (exact integer flip-graph walk from %s, seed %llu).\n",
          from_desc, seed);
  fprintf(f, "# Rows: U (A-blocks row-major), blank, V, blank, W.  Exact by tests/test_oracle_algebra.py.\n");
  fprintf(f, "%d %d %d %zu exact\n", pr.M, pr.K, pr.N, t.size());
  for (int s = 0; s < 3; ++s) {
    for (int i = 0; i < pr.dim(s); ++i) {
      for (size_t r = 0; r < t.size(); ++r) fprintf(f, "%s%d", r ? " " : "", entry(t[r].f[s], i));
      fprintf(f, "\n");
    }
    if (s < 2) fprintf(f, "\n");
  }
  fclose(f);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 5) {
    fprintf(stderr, "usage: %s M K N TARGET [--seed S] [--plateau P] [--seconds T] [--out FILE] [--from FILE] [--best FILE]\n", argv[0]);
    return 2;
  }
  Problem pr{atoi(argv[1]), atoi(argv[2]), atoi(argv[3])};
  const size_t target = (size_t)atoi(argv[4]);
  unsigned long long seed = 1, plateau = 100000;
  double seconds = 600;
  const char* out = nullptr;
  const char* from = nullptr;
  const char* best_out = nullptr;  // --best FILE: rewritten at every new best rank
  for (int i = 5; i + 1 < argc; i += 2) {
    if (!strcmp(argv[i], "--seed")) seed = strtoull(argv[i + 1], nullptr, 10);
    else if (!strcmp(argv[i], "--plateau")) plateau = strtoull(argv[i + 1], nullptr, 10);
    else if (!strcmp(argv[i], "--seconds")) seconds = atof(argv[i + 1]);
    else if (!strcmp(argv[i], "--out")) out = argv[i + 1];
    else if (!strcmp(argv[i], "--from")) from = argv[i + 1];
    else if (!strcmp(argv[i], "--best")) best_out = argv[i + 1];
  }
  if (pr.dim(0) > MAXD || pr.dim(1) > MAXD || pr.dim(2) > MAXD) {
    fprintf(stderr, "dimensions too large\n");
    return 2;
  }
  Walker w{pr, from ? read_file(from, pr) : classical(pr), std::mt19937_64(seed)};
  if (!verify(pr, w.t)) {
    fprintf(stderr, "the starting scheme is not exact\n");
    return 2;
  }
  size_t best = w.t.size();
  std::vector<Term> best_t = w.t;
  unsigned long long since = 0, flips = 0;
  const auto t0 = std::chrono::steady_clock::now();
  while (best > target) {
    ++flips;
    long c0, c1;
    if (w.flip(&c0, &c1)) {
      // a reducible pair must involve one of the two modified terms
      bool red = c0 >= 0 && w.try_reduce((size_t)c0);
      if (!red && c1 >= 0 && (size_t)c1 < w.t.size()) red = w.try_reduce((size_t)c1);
    }
    if (w.t.size() < best) {
      best = w.t.size();
      best_t = w.t;
      since = 0;
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      fprintf(stderr, "rank %zu after %llu flips, %.1f s\n", best, flips, el);
      if (best_out && verify(pr, best_t)) write_file(best_out, pr, best_t, seed, from ? from : "the classical algorithm");
    } else if (++since > plateau) {
      // plateau: restart from the best scheme found, then escape with a rank + 1 move
      w.t = best_t;
      for (int tries = 0; tries < 100 && !w.plus(); ++tries) {
      }
      since = 0;
    }
    if ((flips & 0xFFFFF) == 0) {
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > seconds) break;
    }
  }
  if (!verify(pr, best_t)) {
    fprintf(stderr, "internal error: the scheme is not exact\n");
    return 1;
  }
  fprintf(stderr, "best rank %zu (target %zu), exact\n", best, target);
  if (out && best <= target) write_file(out, pr, best_t, seed, from ? from : "the classical algorithm");
  return best <= target ? 0 : 3;
}
