// K1 / K3: addition-chain kernels, generated per algorithm and compiled with NVRTC for sm_100a.
//
// The paper's code generator emits one specialised C++ routine per algorithm (Sec. 3.1,
// P:547-583) with three addition-chain variants (Sec. 3.2) and optional greedy
// length-two common-subexpression elimination (Sec. 3.3).  Here the planner does the
// same at plan-creation time for the GPU: from a coefficient matrix (outputs x inputs) it emits a
// CUDA kernel in which every S_r / T_r (or C_k) chain is straight-line code, and compiles it with
// NVRTC to an sm_100a cubin (loaded with cudaLibraryLoadData).
//
//  * STREAMING: one thread per element position (x2 with 16-byte vectors) loads each
//    input block element once and writes every output; CSE temporaries live in registers, which
//    is why CSE is free here.
//  * WRITE-ONCE: blockIdx.z selects one output; its thread loads only that chain's
//    inputs and writes one output stream.  Chains are summed in ascending input order (no CSE).
//
// Chain arithmetic: the first nonzero term initialises (copy / negate / scale), later terms add,
// subtract or add a scaled term, compiled with --fmad=false; without CSE this is the oracle's
// order and rounding exactly, so the kernel output is bit-identical to oracle/oracle.c's S_r.
#include <nvrtc.h>

#include <algorithm>
#include <cmath>
#include <functional>
#include <map>
#include <mutex>
#include <set>
#include <sstream>
#include <tuple>

#include "fmm_internal.h"

namespace fmm {

struct LincombKernel {
  LincombSpec spec;
  std::string source;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  int threads = 128;
  LincombCost cost{};
  int temps = 0;
};

size_t lincomb_node_bytes(int nin, int nout) { return sizeof(void*) * (size_t)(nin + nout) + 2 * sizeof(long long); }

namespace {

// A linear expression over variables (inputs 0..nin-1, temporaries nin..).
using Expr = std::map<int, double>;

struct Program {
  int nin = 0;
  std::vector<std::tuple<int, int, double>> temps;  // t = x_a + ratio * x_b
  std::vector<Expr> outs;
};

// Greedy length-two CSE: repeatedly take the pair (a, b, c_b/c_a) that occurs in the
// most outputs (at least twice), ties broken by the lexicographically smallest (a, b, ratio)
// (SPEC S:249 reading R15), introduce t = x_a + ratio x_b and substitute it.
Program build_program(const LincombSpec& s) {
  Program p;
  p.nin = s.nin;
  p.outs.resize(s.nout);
  for (int o = 0; o < s.nout; ++o)
    for (int i = 0; i < s.nin; ++i)
      if (s.coef[o * s.nin + i] != 0.0) p.outs[o][i] = s.coef[o * s.nin + i];
  if (!s.cse || s.strategy != FMM_ADD_STREAMING) return p;
  int next = s.nin;
  for (;;) {
    std::map<std::tuple<int, int, double>, int> count;
    for (const auto& e : p.outs) {
      for (auto a = e.begin(); a != e.end(); ++a)
        for (auto b = std::next(a); b != e.end(); ++b) ++count[{a->first, b->first, b->second / a->second}];
    }
    std::tuple<int, int, double> best;
    int bestc = 1;
    for (const auto& kv : count)
      if (kv.second > bestc) bestc = kv.second, best = kv.first;  // map order = lexicographic tie-break
    if (bestc < 2) break;
    const int a = std::get<0>(best), b = std::get<1>(best);
    const double ratio = std::get<2>(best);
    const int t = next++;
    p.temps.emplace_back(a, b, ratio);
    for (auto& e : p.outs) {
      auto ia = e.find(a), ib = e.find(b);
      if (ia == e.end() || ib == e.end() || ib->second / ia->second != ratio) continue;
      const double ca = ia->second;
      e.erase(ia);
      e.erase(e.find(b));
      e[t] = ca;
    }
  }
  return p;
}

std::string dlit(double c) {
  std::ostringstream ss;
  ss.precision(17);
  ss << c;
  std::string r = ss.str();
  if (r.find('.') == std::string::npos && r.find('e') == std::string::npos) r += ".0";
  return r;
}

// Emit "dst = chain" for one component (suffix "" for scalars, ".x"/".y" for double2).
void emit_chain(std::ostringstream& o, const std::string& dst, const Expr& e, const std::string& comp,
                const std::function<std::string(int)>& var) {
  bool first = true;
  if (e.empty()) {
    o << "    " << dst << comp << " = 0.0;\n";
    return;
  }
  for (const auto& kv : e) {  // ascending variable index
    const std::string v = var(kv.first) + comp;
    const double c = kv.second;
    if (first) {
      if (c == 1.0) o << "    " << dst << comp << " = " << v << ";\n";
      else if (c == -1.0) o << "    " << dst << comp << " = -" << v << ";\n";
      else o << "    " << dst << comp << " = " << dlit(c) << " * " << v << ";\n";
      first = false;
    } else {
      if (c == 1.0) o << "    " << dst << comp << " = " << dst << comp << " + " << v << ";\n";
      else if (c == -1.0) o << "    " << dst << comp << " = " << dst << comp << " - " << v << ";\n";
      else o << "    " << dst << comp << " = " << dst << comp << " + " << dlit(c) << " * " << v << ";\n";
    }
  }
}

std::string generate(const LincombSpec& s, const Program& p, LincombCost& cost) {
  const int nin = s.nin, nout = s.nout, V = s.vec;
  const std::string T = V == 2 ? "double2" : "double";
  std::vector<std::string> comps = V == 2 ? std::vector<std::string>{".x", ".y"} : std::vector<std::string>{""};
  std::ostringstream o;
  o << "// generated by fmm_codegen.cpp: nin=" << nin << " nout=" << nout << " vec=" << V
    << " strategy=" << (s.strategy == FMM_ADD_STREAMING ? "streaming" : "write_once") << " cse=" << s.cse << "\n";
  o << "struct Node { const double* in[" << nin << "]; double* out[" << nout << "]; long long ld_in; long long ld_out; };\n";
  o << "extern \"C\" __global__ void __launch_bounds__(128) lincomb(const Node* __restrict__ nodes, int rows, int cvec) {\n";
  const bool wo = s.strategy == FMM_ADD_WRITE_ONCE;
  if (wo) o << "  const int z = blockIdx.z / " << nout << ", oi = blockIdx.z % " << nout << ";\n";
  else o << "  const int z = blockIdx.z;\n";
  o << "  const Node& nd = nodes[z];\n";
  o << "  const int cv = blockIdx.x * blockDim.x + threadIdx.x;\n";
  o << "  if (cv >= cvec) return;\n";
  o << "  for (int row = blockIdx.y; row < rows; row += gridDim.y) {\n";
  o << "    const long long pi = (long long)row * nd.ld_in + (long long)cv * " << V << ";\n";
  o << "    const long long po = (long long)row * nd.ld_out + (long long)cv * " << V << ";\n";
  auto var = [&](int v) { return v < nin ? "x" + std::to_string(v) : "t" + std::to_string(v - nin); };
  std::set<int> used;
  for (const auto& e : p.outs)
    for (const auto& kv : e)
      if (kv.first < nin) used.insert(kv.first);
  for (const auto& t : p.temps) used.insert(std::get<0>(t) < nin ? std::get<0>(t) : -1), used.insert(std::get<1>(t) < nin ? std::get<1>(t) : -1);
  used.erase(-1);
  double adds = 0, reads = 0, writes = 0;
  if (!wo) {
    for (int i : used) o << "    const " << T << " x" << i << " = __ldg((const " << T << "*)(nd.in[" << i << "] + pi));\n";
    reads = (double)used.size();
    for (size_t t = 0; t < p.temps.size(); ++t) {
      const int a = std::get<0>(p.temps[t]), b = std::get<1>(p.temps[t]);
      const double r = std::get<2>(p.temps[t]);
      o << "    " << T << " t" << t << ";\n";
      for (auto& c : comps) {
        if (r == 1.0) o << "    t" << t << c << " = " << var(a) << c << " + " << var(b) << c << ";\n";
        else if (r == -1.0) o << "    t" << t << c << " = " << var(a) << c << " - " << var(b) << c << ";\n";
        else o << "    t" << t << c << " = " << var(a) << c << " + " << dlit(r) << " * " << var(b) << c << ";\n";
      }
      adds += 1;
    }
    for (int q = 0; q < nout; ++q) {
      o << "    if (nd.out[" << q << "]) {\n    " << T << " y;\n";
      for (auto& c : comps) emit_chain(o, "y", p.outs[q], c, var);
      o << "    *(" << T << "*)(nd.out[" << q << "] + po) = y;\n    }\n";
      adds += p.outs[q].empty() ? 0 : (double)p.outs[q].size() - 1;
      writes += 1;
    }
  } else {
    o << "    switch (oi) {\n";
    for (int q = 0; q < nout; ++q) {
      o << "    case " << q << ": {\n";
      for (const auto& kv : p.outs[q])
        o << "    const " << T << " x" << kv.first << " = __ldg((const " << T << "*)(nd.in[" << kv.first << "] + pi));\n";
      o << "    " << T << " y;\n";
      for (auto& c : comps) emit_chain(o, "y", p.outs[q], c, var);
      o << "    if (nd.out[" << q << "]) *(" << T << "*)(nd.out[" << q << "] + po) = y;\n    } break;\n";
      reads += (double)p.outs[q].size();
      adds += p.outs[q].empty() ? 0 : (double)p.outs[q].size() - 1;
      writes += 1;
    }
    o << "    }\n";
  }
  o << "  }\n}\n";
  cost.adds_per_elem = adds;
  cost.reads_per_elem = reads;
  cost.writes_per_elem = writes;
  return o.str();
}

#define NVRTC_CHECK(x)                                                                         \
  do {                                                                                         \
    nvrtcResult r_ = (x);                                                                      \
    if (r_ != NVRTC_SUCCESS) throw Error(FMM_E_CUDA, std::string("NVRTC: ") + nvrtcGetErrorString(r_)); \
  } while (0)

void compile(LincombKernel& k) {
  nvrtcProgram prog;
  NVRTC_CHECK(nvrtcCreateProgram(&prog, k.source.c_str(), "fmm_lincomb.cu", 0, nullptr, nullptr));
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "--fmad=false", "-lineinfo"};
  nvrtcResult r = nvrtcCompileProgram(prog, 4, opts);
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    throw Error(FMM_E_CUDA, "NVRTC compile failed: " + log);
  }
  size_t n = 0;
  NVRTC_CHECK(nvrtcGetCUBINSize(prog, &n));
  std::vector<char> cubin(n);
  NVRTC_CHECK(nvrtcGetCUBIN(prog, cubin.data()));
  nvrtcDestroyProgram(&prog);
  FMM_CUDA(cudaLibraryLoadData(&k.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
  FMM_CUDA(cudaLibraryGetKernel(&k.kern, k.lib, "lincomb"));
}

std::mutex g_mu;
std::map<std::string, std::shared_ptr<LincombKernel>> g_cache;

}  // namespace

std::shared_ptr<LincombKernel> lincomb_get(const LincombSpec& spec) {
  if (spec.nin < 1 || spec.nout < 1 || (int)spec.coef.size() != spec.nin * spec.nout)
    throw Error(FMM_E_INVALID_ARG, "bad linear-combination spec");
  auto k = std::make_shared<LincombKernel>();
  k->spec = spec;
  Program p = build_program(spec);
  k->temps = (int)p.temps.size();
  k->source = generate(spec, p, k->cost);
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_cache.find(k->source);
  if (it != g_cache.end()) return it->second;
  compile(*k);
  g_cache[k->source] = k;
  return k;
}

void lincomb_launch(const LincombKernel& k, const void* d_nodes, int nnodes, long long rows, long long cols,
                    cudaStream_t stream) {
  if (nnodes <= 0 || rows <= 0 || cols <= 0) return;
  const long long cvec = cols / k.spec.vec;
  if (cvec * k.spec.vec != cols) throw Error(FMM_E_INVALID_ARG, "lincomb: cols not a multiple of vec");
  const long long zdim = (long long)nnodes * (k.spec.strategy == FMM_ADD_WRITE_ONCE ? k.spec.nout : 1);
  if (zdim > 65535) throw Error(FMM_E_UNSUPPORTED, "lincomb: too many nodes in one launch");
  dim3 grid((unsigned)((cvec + k.threads - 1) / k.threads), (unsigned)std::min<long long>(rows, 65535),
            (unsigned)zdim);
  int r = (int)rows, c = (int)cvec;
  void* args[] = {(void*)&d_nodes, &r, &c};
  FMM_CUDA(cudaLaunchKernel((const void*)k.kern, grid, dim3(k.threads), args, 0, stream));
}

LincombCost lincomb_cost(const LincombKernel& k) { return k.cost; }
int lincomb_cse_temps(const LincombKernel& k) { return k.temps; }
std::string lincomb_source(const LincombKernel& k) { return k.source; }

}  // namespace fmm
