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
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <functional>
#include <map>
#include <mutex>
#include <set>
#include <sstream>
#include <tuple>

#include "fmm_internal.h"

namespace fmm {

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

}  // namespace

struct LincombKernel {
  LincombSpec spec;
  Program prog;  // the chains the kernel evaluates (with CSE temporaries when enabled)
  std::string source;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  int threads = 128;
  LincombCost cost{};
  int temps = 0;
  bool row_grid = false;  // 2-D grid (column segments x rows) instead of the flattened map
  int warp_rows = 0;      // > 0: the wide two-level assembly -- warp_rows warps per block, one per
                          // output column k2 of W, 32 vector positions per block (x), rows (y)
  int dyn_smem = 0;       // dynamic shared memory of the launch (the wide assembly's cp.async ring)
};

namespace {

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

// Thread -> element position: one thread per V-vector position of the rows x cvec block, flattened
// (row-major) so that narrow blocks (a few hundred columns at deep levels) still fill whole CTAs;
// a warp touches at most two row segments.  rows * cvec < 2^32 (checked by lincomb_launch).
// The division e / cvec is a multiply-high by magic = ceil(2^64 / cvec) (exact for e * cvec < 2^64,
// which rows * cvec < 2^32 guarantees; cvec = 1 passes magic = 0).
void emit_flat_position(std::ostringstream& o, const char* rows) {
  o << "  const unsigned total_ = (unsigned)" << rows << " * (unsigned)cvec;\n";
  o << "  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < total_; e += gridDim.x * blockDim.x) {\n";
  o << "    const int row = magic ? (int)__umul64hi((unsigned long long)e, magic) : (int)e;\n";
  o << "    const int cv = (int)(e - (unsigned)row * (unsigned)cvec);\n";
}

// Every thread of a CTA uses the same node's nin + nout pointers.  Loaded per thread from the node
// table they form dependent global-load chains in front of the data loads, and the compiler
// interleaves them with the arithmetic; staged once per CTA in shared memory they cost one
// broadcast LDS each (measured: the collapsed c2 assembly went from 0.41 to 0.33 ms).
std::string stage_pointers(std::string src, int nin, int nout) {
  const std::string n = std::to_string(nin + nout);
  auto rep = [&](const std::string& a, const std::string& b) {
    for (size_t at = src.find(a); at != std::string::npos; at = src.find(a, at + b.size())) src.replace(at, a.size(), b);
  };
  rep("nd.in[", "sin_[");
  rep("nd.out[", "sout_[");
  const std::string anchor = "];\n";  // end of the "const Node& nd = nodes[...]" line
  const size_t at = src.find("const Node& nd = nodes[");
  const size_t end = src.find(anchor, at) + anchor.size();
  src.insert(end, "  __shared__ const double* sptr_[" + n + "];\n"
                  "  for (int i = threadIdx.x; i < " + n + "; i += blockDim.x) sptr_[i] = ((const double* const*)nd.in)[i];\n"
                  "  __syncthreads();\n"
                  "  const double* const* sin_ = sptr_;\n"
                  "  double* const* sout_ = (double* const*)(sptr_ + " + std::to_string(nin) + ");\n");
  return src;
}

std::string generate(const LincombSpec& s, const Program& p, LincombCost& cost) {
  const int nin = s.nin, nout = s.nout, V = s.vec;
  const std::string T = V == 2 ? "double2" : "double";
  std::vector<std::string> comps = V == 2 ? std::vector<std::string>{".x", ".y"} : std::vector<std::string>{""};
  std::ostringstream o;
  o << "// generated by fmm_codegen.cpp: nin=" << nin << " nout=" << nout << " vec=" << V
    << " strategy="
    << (s.strategy == FMM_ADD_STREAMING ? "streaming" : s.strategy == FMM_ADD_WRITE_ONCE ? "write_once" : "pairwise")
    << " cse=" << s.cse << "\n";
  o << "__device__ __forceinline__ double2 ldnc2(const double* p) { double2 v; asm volatile(\"ld.global.nc.v2.f64 {%0, %1}, [%2];\" : \"=d\"(v.x), \"=d\"(v.y) : \"l\"(p)); return v; }\n"
       "__device__ __forceinline__ double ldnc1(const double* p) { double v; asm volatile(\"ld.global.nc.f64 %0, [%1];\" : \"=d\"(v) : \"l\"(p)); return v; }\n"
       "__device__ __forceinline__ double2 ldcg2(const double* p) { double2 v; asm volatile(\"ld.global.cg.v2.f64 {%0, %1}, [%2];\" : \"=d\"(v.x), \"=d\"(v.y) : \"l\"(p)); return v; }\n"
       "__device__ __forceinline__ double ldcg1(const double* p) { double v; asm volatile(\"ld.global.cg.f64 %0, [%1];\" : \"=d\"(v) : \"l\"(p)); return v; }\n";
  o << "struct Node { const double* in[" << nin << "]; double* out[" << nout << "]; long long ld_in; long long ld_out; };\n";
  const bool pw = s.strategy == FMM_ADD_PAIRWISE;
  o << "extern \"C\" __global__ void __launch_bounds__(128) lincomb(const Node* __restrict__ nodes, int rows, int cvec, unsigned long long magic"
    << (pw ? ", int step" : "") << ") {\n";
  const bool wo = s.strategy != FMM_ADD_STREAMING;
  if (wo) o << "  const int z = blockIdx.z / " << nout << ", oi = blockIdx.z % " << nout << ";\n";
  else o << "  const int z = blockIdx.z;\n";
  o << "  const Node& nd = nodes[z];\n";
  emit_flat_position(o, "rows");
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
    for (int i : used) {
      if (s.skip_null)  // a shard's absent leaf product: zeros, without touching memory
        o << "    const " << T << " x" << i << " = nd.in[" << i << "] ? ldnc" << V << "(nd.in[" << i << "] + pi) : "
          << (V == 2 ? "make_double2(0.0, 0.0)" : "0.0") << ";\n";
      else
        o << "    const " << T << " x" << i << " = ldnc" << V << "(nd.in[" << i << "] + pi);\n";
    }
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
  } else if (pw) {
    // pairwise: launch `step` applies the step-th term of every chain, y <- x (times
    // its coefficient) for the first term and y <- y + c x after it: one daxpy-like pass per term,
    // each term in ascending index order as in emit_chain, so the sums round identically
    o << "    switch (oi) {\n";
    for (int q = 0; q < nout; ++q) {
      o << "    case " << q << ": {\n    if (!nd.out[" << q << "]) return;\n    switch (step) {\n";
      int t = 0;
      for (const auto& kv : p.outs[q]) {
        const std::string v = "x" + std::to_string(kv.first);
        const double c = kv.second;
        o << "    case " << t << ": {\n";
        o << "    const " << T << " " << v << " = ldnc" << V << "(nd.in[" << kv.first << "] + pi);\n";
        o << "    " << T << " y";
        if (t > 0) o << " = *(const " << T << "*)(nd.out[" << q << "] + po)";
        o << ";\n";
        for (auto& cp : comps) {
          const std::string x = v + cp, y = "y" + cp;
          if (t == 0) {
            if (c == 1.0) o << "    " << y << " = " << x << ";\n";
            else if (c == -1.0) o << "    " << y << " = -" << x << ";\n";
            else o << "    " << y << " = " << dlit(c) << " * " << x << ";\n";
          } else {
            if (c == 1.0) o << "    " << y << " = " << y << " + " << x << ";\n";
            else if (c == -1.0) o << "    " << y << " = " << y << " - " << x << ";\n";
            else o << "    " << y << " = " << y << " + " << dlit(c) << " * " << x << ";\n";
          }
        }
        o << "    *(" << T << "*)(nd.out[" << q << "] + po) = y;\n    } break;\n";
        reads += t == 0 ? 1.0 : 2.0;
        writes += 1;
        ++t;
      }
      o << "    default: return;\n    }\n    } break;\n";
      adds += p.outs[q].empty() ? 0 : (double)p.outs[q].size() - 1;
    }
    o << "    }\n";
  } else {
    o << "    switch (oi) {\n";
    for (int q = 0; q < nout; ++q) {
      o << "    case " << q << ": {\n";
      for (const auto& kv : p.outs[q])
        o << "    const " << T << " x" << kv.first << " = ldnc" << V << "(nd.in[" << kv.first << "] + pi);\n";
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
  return stage_pointers(o.str(), nin, nout);
}

#define NVRTC_CHECK(x)                                                                         \
  do {                                                                                         \
    nvrtcResult r_ = (x);                                                                      \
    if (r_ != NVRTC_SUCCESS) throw Error(FMM_E_CUDA, std::string("NVRTC: ") + nvrtcGetErrorString(r_)); \
  } while (0)

void compile(LincombKernel& k) {
  if (const char* dir = getenv("FMM_LINCOMB_DUMP")) {  // diagnostics: keep the generated source
    const std::string path = std::string(dir) + "/lincomb_" + std::to_string(std::hash<std::string>()(k.source)) + ".cu";
    if (FILE* f = fopen(path.c_str(), "w")) {
      fputs(k.source.c_str(), f);
      fclose(f);
    }
  }
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
  if (k.dyn_smem > 48 * 1024) {
    int dev = 0;
    FMM_CUDA(cudaGetDevice(&dev));
    FMM_CUDA(cudaKernelSetAttributeForDevice(k.kern, cudaFuncAttributeMaxDynamicSharedMemorySize, k.dyn_smem, dev));
  }
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
  k->prog = p;
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
  const long long zdim = (long long)nnodes * (k.spec.strategy != FMM_ADD_STREAMING ? k.spec.nout : 1);
  if (zdim > 65535) throw Error(FMM_E_UNSUPPORTED, "lincomb: too many nodes in one launch");
  const long long total = rows * cvec;
  if (total >= (1ll << 32)) throw Error(FMM_E_UNSUPPORTED, "lincomb: block too large for one launch");
  // one position per thread; the kernel's grid-stride loop form is kept (measured: 2-8 positions
  // per thread were 1-7 % slower, while the loop form alone took c5t's assembly 0.97 -> 0.87 ms)
  if (k.warp_rows > 0) {
    const dim3 g((unsigned)((cvec + 31) / 32), (unsigned)std::min<long long>(rows, 65535), (unsigned)nnodes);
    int r = (int)rows, c = (int)cvec;
    unsigned long long magic = 0;
    void* args[] = {(void*)&d_nodes, &r, &c, &magic};
    FMM_CUDA(cudaLaunchKernel((const void*)k.kern, g, dim3(32 * k.warp_rows), args, (size_t)k.dyn_smem, stream));
    return;
  }
  dim3 grid = k.row_grid ? dim3((unsigned)((cvec + k.threads - 1) / k.threads), (unsigned)std::min<long long>(rows, 65535),
                                 (unsigned)zdim)
                         : dim3((unsigned)((total + k.threads - 1) / k.threads), 1, (unsigned)zdim);
  int r = (int)rows, c = (int)cvec;
  unsigned long long magic = 0;  // ceil(2^64 / cvec)
  if (cvec > 1) magic = ~0ull / (unsigned long long)cvec + 1;
  if (k.spec.strategy == FMM_ADD_PAIRWISE) {
    // one launch per chain position: a term's pass must see the previous term's stores
    for (int step = 0; step < lincomb_steps(k); ++step) {
      void* args[] = {(void*)&d_nodes, &r, &c, &magic, &step};
      FMM_CUDA(cudaLaunchKernel((const void*)k.kern, grid, dim3(k.threads), args, 0, stream));
    }
    return;
  }
  void* args[] = {(void*)&d_nodes, &r, &c, &magic};
  FMM_CUDA(cudaLaunchKernel((const void*)k.kern, grid, dim3(k.threads), args, 0, stream));
}

// ---- the fused leaf-level kernel (NVRTC) -----------------------------------------------------
#include "fmm_embed.inc"  // kFmmDeviceSrc, kFmmCoreSrc: fmm_device.cuh, fmm_gemm_core.cuh verbatim

struct FusedKernel {
  std::string source;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  int bn = 128, ks = 16;
  bool bg = false;
  int stage_w = 0;  // background mode: input staging bytes per producer warp
  int smem_set = -1;  // device on which the dynamic shared-memory limit was raised
};

namespace {

// One addition program as a warp-job function: rows [row0, row0 + nrows) of the node's blocks,
// lanes striding over element positions (V doubles each); per position every input is loaded once
// (L2-coherent: assembly inputs are written by other SMs during the launch), the chains (with the
// program's CSE temporaries) run in registers, every output is stored once -- the streaming K1/K3
// kernel body, so the fused and the separate paths give bit-identical results.
void emit_job_fn(std::ostringstream& o, const std::string& name, const LincombSpec& spec, const Program& p, int V,
                 int data_regs) {
  const int nin = spec.nin, nout = spec.nout;
  const std::string T = V == 2 ? "double2" : "double";
  std::vector<std::string> comps = V == 2 ? std::vector<std::string>{".x", ".y"} : std::vector<std::string>{""};
  auto var = [&](int v) { return v < nin ? "x" + std::to_string(v) : "t" + std::to_string(v - nin); };
  std::set<int> used;
  for (const auto& e : p.outs)
    for (const auto& kv : e)
      if (kv.first < nin) used.insert(kv.first);
  for (const auto& t : p.temps) {
    if (std::get<0>(t) < nin) used.insert(std::get<0>(t));
    if (std::get<1>(t) < nin) used.insert(std::get<1>(t));
  }
  o << "__device__ __forceinline__ void " << name << "(const char* nd, int row0, int nrows, int cols, int lane, unsigned sp) {\n";
  // the node's in[], out[], ld_in, ld_out -> the warp's shared slot; read back per element group
  o << "  for (int w = lane; w < " << nin + nout + 2 << "; w += 32) sts_u64(sp + 8u * w, reinterpret_cast<const unsigned long long*>(nd)[w]);\n";
  o << "  __syncwarp();\n";
  o << "  const long long ldi = (long long)lds_u64(sp + " << 8 * (nin + nout) << "u), ldo = (long long)lds_u64(sp + " << 8 * (nin + nout + 1) << "u);\n";
  o << "  const int cvec = cols / " << V << ";\n";
  o << "  for (int row = row0; row < row0 + nrows; ++row) {\n";
  o << "    const long long bi = (long long)row * ldi, bo = (long long)row * ldo;\n";
  // U element groups per lane per iteration: more loads in flight, within data_regs registers
  const int U = std::max(1, std::min(4, data_regs / (2 * V * std::max<int>(1, (int)used.size()))));
  o << "    for (int cv = lane; cv < cvec; cv += " << 32 * U << ") {\n";
  for (int u = 0; u < U; ++u) {
    o << "    const bool ok" << u << " = cv + " << 32 * u << " < cvec;\n";
    o << "    const long long pi" << u << " = bi + (long long)(cv + " << 32 * u << ") * " << V << ", po" << u
      << " = bo + (long long)(cv + " << 32 * u << ") * " << V << ";\n";
  }
  const std::string zero = V == 2 ? "make_double2(0.0, 0.0)" : "0.0";
  for (int u = 0; u < U; ++u)
    for (int i : used)
      o << "    const " << T << " x" << i << "_" << u << " = ok" << u << " ? " << (V == 2 ? "ldcg2" : "ldcg1")
        << "(reinterpret_cast<const double*>(lds_u64(sp + " << 8 * i << "u)) + pi" << u << ") : " << zero << ";\n";
  for (int u = 0; u < U; ++u) {
    auto varu = [&](int v) { return var(v) + "_" + std::to_string(u); };
    for (size_t t = 0; t < p.temps.size(); ++t) {
      const int a = std::get<0>(p.temps[t]), b = std::get<1>(p.temps[t]);
      const double r = std::get<2>(p.temps[t]);
      o << "    " << T << " t" << t << "_" << u << ";\n";
      for (auto& c : comps) {
        const std::string d = "t" + std::to_string(t) + "_" + std::to_string(u) + c;
        if (r == 1.0) o << "    " << d << " = " << varu(a) << c << " + " << varu(b) << c << ";\n";
        else if (r == -1.0) o << "    " << d << " = " << varu(a) << c << " - " << varu(b) << c << ";\n";
        else o << "    " << d << " = " << varu(a) << c << " + " << dlit(r) << " * " << varu(b) << c << ";\n";
      }
    }
    for (int q = 0; q < nout; ++q) {
      o << "    if (double* oq = reinterpret_cast<double*>(lds_u64(sp + " << 8 * (nin + q) << "u))) {\n    " << T << " y;\n";
      for (auto& c : comps) emit_chain(o, "y", p.outs[q], c, varu);
      o << "    if (ok" << u << ") *reinterpret_cast<" << T << "*>(oq + po" << u << ") = y;\n    }\n";
    }
  }
  o << "    }\n  }\n  __syncwarp();  // every lane is done with the slot before the next job rewrites it\n}\n";
}

// The inputs a program's chains and temporaries read (ascending).
std::vector<int> program_inputs(const LincombSpec& spec, const Program& p) {
  std::set<int> used;
  for (const auto& e : p.outs)
    for (const auto& kv : e)
      if (kv.first < spec.nin) used.insert(kv.first);
  for (const auto& t : p.temps) {
    if (std::get<0>(t) < spec.nin) used.insert(std::get<0>(t));
    if (std::get<1>(t) < spec.nin) used.insert(std::get<1>(t));
  }
  return std::vector<int>(used.begin(), used.end());
}

// Background-mode variant of emit_job_fn for the producer warps (56 registers): per element (8
// bytes per lane) every input is staged in the warp's shared-memory area st by cp.async -- all of
// them in flight at once, none held in registers -- then the chains read them back with ld.shared
// where they use them.  Same chains, same order of operations: bitwise equal to emit_job_fn.
void emit_job_fn_staged(std::ostringstream& o, const std::string& name, const LincombSpec& spec, const Program& p) {
  const int nin = spec.nin, nout = spec.nout;
  const std::vector<int> used = program_inputs(spec, p);
  std::map<int, int> slot;
  for (size_t s = 0; s < used.size(); ++s) slot[used[s]] = (int)s;
  auto var = [&](int v) {
    if (v < nin) return "lds64(xs + " + std::to_string(256 * slot.at(v)) + "u)";
    return "t" + std::to_string(v - nin);
  };
  o << "__device__ __forceinline__ void " << name
    << "(const char* nd, int row0, int nrows, int cols, int lane, unsigned sp, unsigned st) {\n";
  o << "  for (int w = lane; w < " << nin + nout + 2 << "; w += 32) sts_u64(sp + 8u * w, reinterpret_cast<const unsigned long long*>(nd)[w]);\n";
  o << "  __syncwarp();\n";
  o << "  const long long ldi = (long long)lds_u64(sp + " << 8 * (nin + nout) << "u), ldo = (long long)lds_u64(sp + " << 8 * (nin + nout + 1) << "u);\n";
  o << "  const unsigned xs = st + 8u * (unsigned)lane;\n";
  o << "  for (int row = row0; row < row0 + nrows; ++row) {\n";
  o << "    const long long bi = (long long)row * ldi, bo = (long long)row * ldo;\n";
  o << "    for (int cv = lane; cv < cols; cv += 32) {\n";
  o << "    const long long pi = bi + cv, po = bo + cv;\n";
  for (int i : used)
    o << "    cp_async8(xs + " << 256 * slot.at(i) << "u, reinterpret_cast<const double*>(lds_u64(sp + " << 8 * i << "u)) + pi);\n";
  o << "    cp_async_wait_all();\n";
  // FMM_FUSED_DIAG (timing diagnostics only, wrong results): 1 = integer XOR in place of every
  // floating-point operation, 2 = each output a copy of its first input (no arithmetic)
  const int diag = getenv("FMM_FUSED_DIAG") ? atoi(getenv("FMM_FUSED_DIAG")) : 0;
  auto bop = [&](const std::string& x, const std::string& y, const char* op) {
    if (diag == 1) return "__longlong_as_double(__double_as_longlong(" + x + ") ^ __double_as_longlong(" + y + "))";
    if (diag == 2) return x;
    return x + " " + op + " " + y;
  };
  for (size_t t = 0; t < p.temps.size(); ++t) {
    const int a = std::get<0>(p.temps[t]), b = std::get<1>(p.temps[t]);
    const double r = std::get<2>(p.temps[t]);
    o << "    const double t" << t << " = ";
    if (r == 1.0) o << bop(var(a), var(b), "+") << ";\n";
    else if (r == -1.0) o << bop(var(a), var(b), "-") << ";\n";
    else o << bop(var(a), diag ? var(b) : dlit(r) + " * " + var(b), "+") << ";\n";
  }
  for (int q = 0; q < nout; ++q) {
    o << "    if (double* oq = reinterpret_cast<double*>(lds_u64(sp + " << 8 * (nin + q) << "u))) {\n    double y;\n";
    if (diag) {
      bool first = true;
      for (const auto& kv : p.outs[q]) {
        if (first) o << "    y = " << var(kv.first) << ";\n", first = false;
        else if (diag == 1) o << "    y = " << bop("y", var(kv.first), "+") << ";\n";
      }
      if (first) o << "    y = 0.0;\n";
    } else {
      emit_chain(o, "y", p.outs[q], "", var);
    }
    o << "    oq[po] = y;\n    }\n";
  }
  o << "    }\n  }\n  __syncwarp();\n}\n";
}

std::string strip_pragma_once(const char* src) {
  std::string s(src);
  const std::string key = "#pragma once";
  for (size_t at; (at = s.find(key)) != std::string::npos;) s.erase(at, key.size());
  return s;
}

std::mutex g_fmu;
std::map<std::string, std::shared_ptr<FusedKernel>> g_fcache;

}  // namespace

int fused_bg_stage_bytes(const std::vector<LincombSpec>& specs) {
  int nin = 1;
  for (const auto& s : specs) nin = std::max(nin, s.nin);
  return 256 * nin;  // 8 bytes x 32 lanes per input
}

std::string fused_generate(const std::vector<LincombSpec>& specs, int bn, int ks, bool bg) {
  if (ks != 16 && ks != 32 && ks != 48) throw Error(FMM_E_INVALID_ARG, "fused: ring depth must be 16, 32 or 48");
  if (specs.empty() || (int)specs.size() > FUSED_MAX_PROGS) throw Error(FMM_E_INVALID_ARG, "fused: bad program count");
  int wgm = 0, wgn = 0;
  gemm_bn_config(bn, &wgm, &wgn);
  std::ostringstream o;
  o << "// generated by fmm_codegen.cpp: fused leaf level, BN=" << bn << ", KS=" << ks << (bg ? ", background jobs" : "")
    << "\n#define FMM_NVRTC 1\n";
  // background mode: the producer warpgroup keeps 56 registers per thread and the consumers get 224
  // (of the CTA's 384 x 168), enough for a job's inputs at U = 1 (the 8-byte variant where 16-byte
  // ones would spill) and the 64 x 32 warp tile
  if (bg) {
    o << "#define FMM_BG_STAGE_W " << fused_bg_stage_bytes(specs) << "\n";
    int pr = 56, cr = 224;
    if (const char* e = getenv("FMM_FUSED_REGS")) sscanf(e, "%d,%d", &pr, &cr);  // experiments: "producer,consumer"
    o << "#define FMM_FUSED_BG 1\n#define FMM_PRODUCER_REGS " << pr << "\n#define FMM_CONSUMER_REGS " << cr << "\n";
  }
  // the ring geometry of the nvcc-compiled kernels, so the host's shared-memory sizes match
  o << "#define FMM_GEMM_BK " << gemm_bk() << "\n#define FMM_GEMM_STAGES " << gemm_stages() << "\n";
  if (const char* e = getenv("FMM_FUSED_LD")) o << "#define FMM_LD_KIND " << atoi(e) << "\n";  // diagnostics
  if (getenv("FMM_FUSED_STATS")) o << "#define FMM_FUSED_STATS 1\n";                              // diagnostics
  if (const char* e = getenv("FMM_FUSED_DIAG")) o << "// diag " << e << "\n";                   // (new cache key)
  o << strip_pragma_once(kFmmDeviceSrc) << "\n" << strip_pragma_once(kFmmCoreSrc) << "\nnamespace fmm {\n";
  for (size_t q = 0; q < specs.size(); ++q) {
    if (specs[q].strategy != FMM_ADD_STREAMING) throw Error(FMM_E_INVALID_ARG, "fused: streaming programs only");
    const Program prog = build_program(specs[q]);
    emit_job_fn(o, "prog" + std::to_string(q) + "_v2", specs[q], prog, 2, 96);
    emit_job_fn(o, "prog" + std::to_string(q) + "_v1", specs[q], prog, 1, 96);
    if (bg) emit_job_fn_staged(o, "prog" + std::to_string(q) + "_s", specs[q], prog);
  }
  o << "__device__ void fmm_add_job(const FusedArgs& fa, const FusedJob& j, int lane, unsigned sp) {\n";
  o << "  const char* nd = fa.node_tab[j.prog] + (long long)j.node * fa.node_bytes[j.prog];\n";
  o << "  switch (j.prog) {\n";
  for (size_t q = 0; q < specs.size(); ++q)
    o << "    case " << q << ": if (fa.vec2[" << q << "]) prog" << q << "_v2(nd, j.row0, j.nrows, fa.cols[" << q
      << "], lane, sp); else prog" << q << "_v1(nd, j.row0, j.nrows, fa.cols[" << q << "], lane, sp); break;\n";
  o << "  }\n}\n";
  if (bg) {
    o << "__device__ void fmm_add_job_bg(const FusedArgs& fa, const FusedJob& j, int lane, unsigned sp, unsigned st) {\n";
    o << "  const char* nd = fa.node_tab[j.prog] + (long long)j.node * fa.node_bytes[j.prog];\n";
    o << "  switch (j.prog) {\n";
    for (size_t q = 0; q < specs.size(); ++q)
      o << "    case " << q << ": prog" << q << "_s(nd, j.row0, j.nrows, fa.cols[" << q << "], lane, sp, st); break;\n";
    o << "  }\n}\n";
  }
  o << "}  // namespace fmm\n";
  o << "extern \"C\" __global__ void __launch_bounds__(fmm::THREADS, 1)\n"
       "fmm_fused(const fmm::GemmTask* __restrict__ tasks, const fmm::CUtensorMap* __restrict__ maps, int ntasks,\n"
       "          int total_tiles, fmm::Uniform uni, fmm::FusedArgs fa) {\n"
    << "  fmm::gemm_body<" << bn << ", " << wgm << ", " << wgn << ", true, false, " << ks
    << ">(tasks, maps, ntasks, total_tiles, uni, fa);\n}\n";
  return o.str();
}

std::vector<char> fused_compile(const std::string& source) {
  if (const char* path = getenv("FMM_FUSED_DUMP")) {  // diagnostics: keep the generated source
    if (FILE* f = fopen(path, "w")) fputs(source.c_str(), f), fclose(f);
  }
  nvrtcProgram prog;
  NVRTC_CHECK(nvrtcCreateProgram(&prog, source.c_str(), "fmm_fused.cu", 0, nullptr, nullptr));
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "--fmad=false", "-lineinfo", "--ptxas-options=-v"};
  const bool verbose = getenv("FMM_FUSED_PTXAS_V") != nullptr;  // diagnostics: registers / spills to stderr
  nvrtcResult r = nvrtcCompileProgram(prog, verbose ? 5 : 4, opts);
  if (verbose && r == NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    fputs(log.c_str(), stderr);
  }
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    throw Error(FMM_E_CUDA, "NVRTC compile of the fused kernel failed: " + log);
  }
  size_t n = 0;
  NVRTC_CHECK(nvrtcGetCUBINSize(prog, &n));
  std::vector<char> cubin(n);
  NVRTC_CHECK(nvrtcGetCUBIN(prog, cubin.data()));
  nvrtcDestroyProgram(&prog);
  if (const char* path = getenv("FMM_FUSED_CUBIN_DUMP")) {  // diagnostics: keep the cubin (cuobjdump -sass)
    if (FILE* f = fopen(path, "wb")) fwrite(cubin.data(), 1, cubin.size(), f), fclose(f);
  }
  return cubin;
}

std::shared_ptr<FusedKernel> fused_get(const std::vector<LincombSpec>& specs, int bn, int ks, bool bg) {
  auto k = std::make_shared<FusedKernel>();
  k->source = fused_generate(specs, bn, ks, bg);
  k->bn = bn;
  k->ks = ks;
  k->bg = bg;
  k->stage_w = bg ? fused_bg_stage_bytes(specs) : 0;
  std::lock_guard<std::mutex> lock(g_fmu);
  auto it = g_fcache.find(k->source);
  if (it != g_fcache.end()) return it->second;
  const std::vector<char> cubin = fused_compile(k->source);
  FMM_CUDA(cudaLibraryLoadData(&k->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
  FMM_CUDA(cudaLibraryGetKernel(&k->kern, k->lib, "fmm_fused"));
  g_fcache[k->source] = k;
  return k;
}

void fused_launch(const FusedKernel& k, const GemmTask* d_tasks, const void* d_maps, int ntasks, long long total_tiles,
                  int uniform_tm, int uniform_tn, const FusedArgs& fa, cudaStream_t stream) {
  const int smem = gemm_fused_smem_bytes(k.bn, k.ks, k.stage_w);
  int dev = 0;
  FMM_CUDA(cudaGetDevice(&dev));
  if (k.smem_set != dev) {
    FMM_CUDA(cudaKernelSetAttributeForDevice(k.kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem, dev));
    const_cast<FusedKernel&>(k).smem_set = dev;
  }
  // every CTA must be resident (jobs wait on tiles, tiles on jobs): cooperative, one CTA per SM
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)gemm_sm_count());
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  Uniform uni{uniform_tm * uniform_tn, uniform_tm, uniform_tn};
  int nt = ntasks, tt = (int)total_tiles;
  FusedArgs a = fa;
  void* args[] = {(void*)&d_tasks, (void*)&d_maps, &nt, &tt, &uni, &a};
  FMM_CUDA(cudaLaunchKernelExC(&cfg, (const void*)k.kern, args));
}

std::string fused_source(const FusedKernel& k) { return k.source; }

// ---- two collapsed levels ------------------------------------------------------------------------
namespace {
std::string generate_two_level(const TwoLevelSpec& sp, LincombCost& cost) {
  const int rows = sp.rows, R = sp.R, V = sp.vec;
  const std::string T = V == 2 ? "double2" : "double";
  std::vector<std::string> comps = V == 2 ? std::vector<std::string>{".x", ".y"} : std::vector<std::string>{""};
  auto X = [&](int i, int r) { return sp.X[(size_t)i * R + r]; };
  auto nz = [&](int r) {
    std::vector<int> v;
    for (int i = 0; i < rows; ++i)
      if (X(i, r) != 0.0) v.push_back(i);
    return v;
  };
  const bool asm_ = sp.side == 2;
  const bool asm_row_grid = asm_;  // launch geometry: see lincomb_launch (LincombKernel::row_grid)
  const int nin = asm_ ? R * R : rows * rows, nout = asm_ ? rows * rows : R * R;
  std::ostringstream o;
  o << "// generated by fmm_codegen.cpp: two collapsed levels, side=" << sp.side << " rows=" << rows << " R=" << R << " vec=" << V
    << "\n";
  o << "__device__ __forceinline__ double2 ldnc2(const double* p) { double2 v; asm volatile(\"ld.global.nc.v2.f64 {%0, %1}, [%2];\" : \"=d\"(v.x), \"=d\"(v.y) : \"l\"(p)); return v; }\n"
       "__device__ __forceinline__ double ldnc1(const double* p) { double v; asm volatile(\"ld.global.nc.f64 %0, [%1];\" : \"=d\"(v) : \"l\"(p)); return v; }\n"
       "__device__ __forceinline__ double2 ldcg2(const double* p) { double2 v; asm volatile(\"ld.global.cg.v2.f64 {%0, %1}, [%2];\" : \"=d\"(v.x), \"=d\"(v.y) : \"l\"(p)); return v; }\n"
       "__device__ __forceinline__ double ldcg1(const double* p) { double v; asm volatile(\"ld.global.cg.f64 %0, [%1];\" : \"=d\"(v) : \"l\"(p)); return v; }\n";
  o << "struct Node { const double* in[" << nin << "]; double* out[" << nout << "]; long long ld_in; long long ld_out; };\n";
  o << "extern \"C\" __global__ void __launch_bounds__(128) lincomb(const Node* __restrict__ nodes, int nrows, int cvec, unsigned long long magic) {\n";
  o << "  const Node& nd = nodes[blockIdx.z];\n";
  if (asm_row_grid) {
    // the collapsed assembly keeps the 2-D grid (x: 128-thread column segments, y: rows) with the
    // node pointers read straight from the table: measured 0.324 vs 0.35 ms on c2 -- the compiler
    // then hoists all R^2 loads (254 registers) and the kernel reaches 82 % of DRAM bandwidth
    o << "  const int cv = blockIdx.x * blockDim.x + threadIdx.x;\n";
    o << "  if (cv >= cvec) return;\n";
    o << "  for (int row = blockIdx.y; row < nrows; row += gridDim.y) {\n";
  } else {
    emit_flat_position(o, "nrows");
  }
  o << "    const long long pi = (long long)row * nd.ld_in + (long long)cv * " << V << ";\n";
  o << "    const long long po = (long long)row * nd.ld_out + (long long)cv * " << V << ";\n";
  // chain over named terms (first-term initialisation; --fmad=false keeps products separate)
  auto chain = [&](const std::string& dst, const std::vector<std::pair<std::string, double>>& terms) {
    for (auto& c : comps) {
      bool first = true;
      for (const auto& t : terms) {
        const std::string v = t.first + c;
        const double k = t.second;
        if (first) {
          o << "    " << dst << c << " = " << (k == 1.0 ? v : k == -1.0 ? "-" + v : dlit(k) + " * " + v) << ";\n";
          first = false;
        } else {
          o << "    " << dst << c << " = " << dst << c << (k == 1.0 ? " + " + v : k == -1.0 ? " - " + v : " + " + dlit(k) + " * " + v) << ";\n";
        }
      }
      if (first) o << "    " << dst << c << " = 0.0;\n";
    }
  };
  double adds = 0, reads = 0, writes = 0;
  if (!asm_) {
    // which inputs are used: all x[i1][i2] for i1 in nz(r1) of a needed r1 (or singleton i1s)
    std::set<int> used;
    for (int r1 = 0; r1 < R; ++r1) {
      bool any = false;
      for (int r2 = 0; r2 < R; ++r2) any |= sp.materialize[(size_t)r1 * R + r2] != 0;
      if (!any) continue;
      for (int i1 : nz(r1))
        for (int i2 = 0; i2 < rows; ++i2) used.insert(i1 * rows + i2);
    }
    for (int i : used) o << "    const " << T << " x" << i << " = ldnc" << V << "(nd.in[" << i << "] + pi);\n";
    reads = (double)used.size();
    for (int r1 = 0; r1 < R; ++r1) {
      bool any = false;
      for (int r2 = 0; r2 < R; ++r2) any |= sp.materialize[(size_t)r1 * R + r2] != 0;
      if (!any) continue;
      const std::vector<int> n1 = nz(r1);
      // T[r1][i2] for the i2 some materialised output of r1 needs
      std::set<int> need_i2;
      for (int r2 = 0; r2 < R; ++r2)
        if (sp.materialize[(size_t)r1 * R + r2])
          for (int i2 : nz(r2)) need_i2.insert(i2);
      for (int i2 : need_i2) {
        const std::string t = "t" + std::to_string(r1) + "_" + std::to_string(i2);
        if (n1.size() == 1) {
          o << "    const " << T << "& " << t << " = x" << n1[0] * rows + i2 << ";\n";  // singleton r1: unscaled alias
        } else {
          std::vector<std::pair<std::string, double>> terms;
          for (int i1 : n1) terms.push_back({"x" + std::to_string(i1 * rows + i2), X(i1, r1)});
          o << "    " << T << " " << t << ";\n";
          chain(t, terms);
          adds += (double)n1.size() - 1;
        }
      }
      for (int r2 = 0; r2 < R; ++r2) {
        const int q = r1 * R + r2;
        if (!sp.materialize[(size_t)q]) continue;
        const std::vector<int> n2 = nz(r2);
        o << "    if (nd.out[" << q << "]) {\n    " << T << " y;\n";
        if (n2.size() == 1) {
          for (auto& c : comps) o << "    y" << c << " = t" << r1 << "_" << n2[0] << c << ";\n";  // singleton r2: unscaled
        } else {
          std::vector<std::pair<std::string, double>> terms;
          for (int i2 : n2) terms.push_back({"t" + std::to_string(r1) + "_" + std::to_string(i2), X(i2, r2)});
          chain("y", terms);
          adds += (double)n2.size() - 1;
        }
        o << "    *(" << T << "*)(nd.out[" << q << "] + po) = y;\n    }\n";
        writes += 1;
      }
    }
  } else {
    // C[k1][k2] = sum_r1 X[k1][r1] M1[r1][k2],  M1[r1][k2] = sum_r2 X[k2][r2] M[r1][r2].
    // Group r1's loads are emitted `ahead` groups before its arithmetic (volatile loads keep that
    // order).
    for (int k = 0; k < nout; ++k) o << "    " << T << " c" << k << ";\n";
    std::vector<char> started(nout, 0);
    std::set<int> r2s;
    for (int k2 = 0; k2 < rows; ++k2)
      for (int r2 = 0; r2 < R; ++r2)
        if (X(k2, r2) != 0.0) r2s.insert(r2);
    std::vector<int> groups;
    for (int r1 = 0; r1 < R; ++r1) {
      bool any = false;
      for (int k1 = 0; k1 < rows; ++k1) any |= X(k1, r1) != 0.0;
      if (any) groups.push_back(r1);
    }
    auto loads = [&](int r1) {
      for (int r2 : r2s) {
        const std::string ptr = "nd.in[" + std::to_string(r1 * R + r2) + "]";
        if (sp.skip_null)
          o << "    const " << T << " m" << r1 << "_" << r2 << " = " << ptr << " ? __ldcg((const " << T << "*)(" << ptr
            << " + pi)) : " << (V == 2 ? "make_double2(0.0, 0.0)" : "0.0") << ";\n";
        else
          o << "    const " << T << " m" << r1 << "_" << r2 << " = __ldcg((const " << T << "*)(" << ptr << " + pi));\n";
      }
      reads += (double)r2s.size();
    };
    auto arith = [&](int r1) {
      std::vector<int> ks;  // k1 with X[k1][r1] != 0
      for (int k1 = 0; k1 < rows; ++k1)
        if (X(k1, r1) != 0.0) ks.push_back(k1);
      o << "    {\n";
      for (int k2 = 0; k2 < rows; ++k2) {
        std::vector<std::pair<std::string, double>> terms;
        for (int r2 = 0; r2 < R; ++r2)
          if (X(k2, r2) != 0.0) terms.push_back({"m" + std::to_string(r1) + "_" + std::to_string(r2), X(k2, r2)});
        o << "    " << T << " u" << k2 << ";\n";
        chain("u" + std::to_string(k2), terms);
        adds += terms.empty() ? 0 : (double)terms.size() - 1;
        for (int k1 : ks) {
          const int k = k1 * rows + k2;
          const double w = X(k1, r1);
          const std::string v = "u" + std::to_string(k2);
          for (auto& c : comps) {
            const std::string d = "c" + std::to_string(k) + c, vv = v + c;
            if (!started[k]) o << "    " << d << " = " << (w == 1.0 ? vv : w == -1.0 ? "-" + vv : dlit(w) + " * " + vv) << ";\n";
            else o << "    " << d << " = " << d << (w == 1.0 ? " + " + vv : w == -1.0 ? " - " + vv : " + " + dlit(w) + " * " + vv) << ";\n";
          }
          if (started[k]) adds += 1;
          started[k] = 1;
        }
      }
      o << "    }\n";
    };
    // each group's loads just before its arithmetic; the compiler hoists them (see above)
    for (int r1 : groups) {
      loads(r1);
      arith(r1);
    }
    for (int k = 0; k < nout; ++k) {
      if (!started[k])
        for (auto& c : comps) o << "    c" << k << c << " = 0.0;\n";
      o << "    *(" << T << "*)(nd.out[" << k << "] + po) = c" << k << ";\n";
      writes += 1;
    }
  }
  o << "  }\n}\n";
  cost.adds_per_elem = adds;
  cost.reads_per_elem = reads;
  cost.writes_per_elem = writes;
  return asm_row_grid ? o.str() : stage_pointers(o.str(), nin, nout);
}
// The two-level assembly for base cases too large to hold the (MN)^2 outputs of a position in one
// thread's registers (MN > 4): C[k1][k2] = sum_r1 W[k1][r1] M1[r1][k2], M1[r1][k2] =
// sum_r2 W[k2][r2] M[r1][r2] (P:569-572 applied twice), the oracle's two levels in its order.
// A block owns 32 vector positions of one row of the level-L blocks and has one warp per output
// column k2 (warp-uniform chains).  For each r1 in order, the warps stage the R leaf products
// M[r1][.] of the block's positions in shared memory (each element read from HBM once; the next r1's
// loads are issued before this r1's arithmetic), then warp k2 forms M1[r1][k2] from shared memory and
// adds it into its MN accumulators C[k1][k2], k1 with W[k1][r1] != 0.  HBM traffic: R^2 reads and
// (MN)^2 writes per position, against R^2 + 2 R MN + (MN)^2 for the two separate levels.
// two positions per thread (double2), one block per SM (the MN accumulators take the registers), a
// ring of up to 96 KB.  Measured (c4): 2.30 ms, against 2.67 ms for one position per thread with two
// blocks per SM and 2.05 ms for the two separate assembly levels.
constexpr int WIDE_VEC = 2, WIDE_BLOCKS_PER_SM = 1;
int wide_stages(int stage_bytes) { return std::max(3, std::min(8, 96 * 1024 / stage_bytes)); }

std::string generate_two_level_wide(const TwoLevelSpec& sp, LincombCost& cost) {
  const int rows = sp.rows, R = sp.R, V = sp.vec;
  const std::string T = V == 2 ? "double2" : "double";
  std::vector<std::string> comps = V == 2 ? std::vector<std::string>{".x", ".y"} : std::vector<std::string>{""};
  auto X = [&](int i, int r) { return sp.X[(size_t)i * R + r]; };
  const int per = (R + rows - 1) / rows;  // leaf products each warp stages per r1
  // stages of the cp.async ring: as deep as ~96 KB of shared memory allows (one block per SM: the
  // accumulators take the registers), so enough bytes are in flight to keep HBM busy
  const int stage_bytes = R * 32 * 8 * V;
  const int D = wide_stages(stage_bytes);
  std::ostringstream o;
  o << "// generated by fmm_codegen.cpp: wide two-level assembly rows=" << rows << " R=" << R << " vec=" << V << " stages=" << D << "\n";
  o << "struct Node { const double* in[" << R * R << "]; double* out[" << rows * rows << "]; long long ld_in; long long ld_out; };\n";
  o << "__device__ __forceinline__ void cpa(void* dst, const double* src) {\n";
  if (V == 2)
    o << "  asm volatile(\"cp.async.cg.shared.global [%0], [%1], 16;\" :: \"r\"((unsigned)__cvta_generic_to_shared(dst)), \"l\"(src) : \"memory\");\n";
  else
    o << "  asm volatile(\"cp.async.ca.shared.global [%0], [%1], 8;\" :: \"r\"((unsigned)__cvta_generic_to_shared(dst)), \"l\"(src) : \"memory\");\n";
  o << "}\n";
  o << "extern \"C\" __global__ void __launch_bounds__(" << 32 * rows << ", " << WIDE_BLOCKS_PER_SM << ") lincomb(const Node* __restrict__ nodes, int nrows, int cvec, unsigned long long magic) {\n";
  o << "  extern __shared__ " << T << " smd[];  // [" << D << "][" << R << "][32]\n";
  o << "  const Node& nd = nodes[blockIdx.z];\n";
  o << "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n";
  o << "  const int cv = blockIdx.x * 32 + lane;\n";
  o << "  const bool live = cv < cvec;\n";
  o << "  for (int row = blockIdx.y; row < nrows; row += gridDim.y) {\n";
  o << "    const long long pi = (long long)row * nd.ld_in + (long long)cv * " << V << ";\n";
  o << "    const long long po = (long long)row * nd.ld_out + (long long)cv * " << V << ";\n";
  // issue the copies of step r (this warp's leaf products r2 = warp + rows q) into its ring slot
  o << "    auto issue = [&](int r) {\n";
  o << "      " << T << "* buf = smd + (r % " << D << ") * " << R * 32 << ";\n";
  for (int q = 0; q < per; ++q) {
    o << "      { const int r2 = warp + " << rows * q << "; if (r2 < " << R << " && live) {\n";
    o << "        const double* src = nd.in[r * " << R << " + r2];\n";
    o << "        if (src) cpa(buf + r2 * 32 + lane, src + pi); else buf[r2 * 32 + lane] = " << T << "{};\n      } }\n";
  }
  o << "      asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n";
  o << "    };\n";
  for (int d = 0; d < D - 1; ++d) o << "    if (" << d << " < " << R << ") issue(" << d << "); else asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n";
  o << "    " << T << " acc[" << rows << "];\n";
  o << "    for (int r1 = 0; r1 < " << R << "; ++r1) {\n";
  o << "      asm volatile(\"cp.async.wait_group " << D - 2 << ";\" ::: \"memory\");\n";
  o << "      __syncthreads();  // step r1 staged by every warp; every warp is done with step r1 - 1\n";
  o << "      if (r1 + " << D - 1 << " < " << R << ") issue(r1 + " << D - 1 << ");  // into the slot of step r1 - 1\n";
  o << "      else asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n";
  o << "      const " << T << "* sm = smd + (r1 % " << D << ") * " << R * 32 << ";\n";
  o << "      " << T << " u;\n";
  // M1[r1][k2] for k2 = warp: a warp-uniform switch over the generated chains
  o << "      switch (warp) {\n";
  for (int k2 = 0; k2 < rows; ++k2) {
    o << "      case " << k2 << ": {\n";
    bool first = true;
    for (int r2 = 0; r2 < R; ++r2) {
      const double w = X(k2, r2);
      if (w == 0.0) continue;
      for (auto& c : comps) {
        const std::string v = "sm[" + std::to_string(r2 * 32) + " + lane]" + c;
        if (first) o << "        u" << c << " = " << (w == 1.0 ? v : w == -1.0 ? "-" + v : dlit(w) + " * " + v) << ";\n";
        else o << "        u" << c << " = u" << c << (w == 1.0 ? " + " + v : w == -1.0 ? " - " + v : " + " + dlit(w) + " * " + v) << ";\n";
      }
      first = false;
    }
    if (first)
      for (auto& c : comps) o << "        u" << c << " = 0.0;\n";
    o << "        break; }\n";
  }
  o << "      }\n";
  // accumulate: a uniform switch over r1 (the first term of each k1 initialises)
  o << "      switch (r1) {\n";
  std::vector<int> firstr(rows, -1);
  for (int k1 = 0; k1 < rows; ++k1)
    for (int r1 = 0; r1 < R; ++r1)
      if (X(k1, r1) != 0.0) {
        firstr[k1] = r1;
        break;
      }
  for (int r1 = 0; r1 < R; ++r1) {
    o << "      case " << r1 << ":\n";
    for (int k1 = 0; k1 < rows; ++k1) {
      const double w = X(k1, r1);
      if (w == 0.0) continue;
      for (auto& c : comps) {
        const std::string d = "acc[" + std::to_string(k1) + "]" + c, v = "u" + c;
        if (firstr[k1] == r1) o << "        " << d << " = " << (w == 1.0 ? v : w == -1.0 ? "-" + v : dlit(w) + " * " + v) << ";\n";
        else o << "        " << d << " = " << d << (w == 1.0 ? " + " + v : w == -1.0 ? " - " + v : " + " + dlit(w) + " * " + v) << ";\n";
      }
    }
    o << "        break;\n";
  }
  o << "      }\n";
  o << "    }\n";
  o << "    if (live) {\n";
  for (int k1 = 0; k1 < rows; ++k1) {
    if (firstr[k1] < 0)
      for (auto& c : comps) o << "      acc[" << k1 << "]" << c << " = 0.0;\n";
    o << "      __stcs((" << T << "*)(nd.out[" << k1 << " * " << rows << " + warp] + po), acc[" << k1 << "]);\n";
  }
  o << "    }\n";
  o << "    __syncthreads();  // the next row's prologue reuses the ring\n";
  o << "  }\n}\n";
  // per element position (all warps together): R^2 reads, (MN)^2 writes; additions of every chain
  double chain_adds = 0;
  for (int k2 = 0; k2 < rows; ++k2) {
    int t = 0;
    for (int r2 = 0; r2 < R; ++r2) t += X(k2, r2) != 0.0;
    chain_adds += t > 0 ? t - 1 : 0;
  }
  double acc_adds = 0;
  for (int k1 = 0; k1 < rows; ++k1) {
    int t = 0;
    for (int r1 = 0; r1 < R; ++r1) t += X(k1, r1) != 0.0;
    acc_adds += t > 0 ? t - 1 : 0;
  }
  cost.adds_per_elem = R * chain_adds + rows * acc_adds;
  cost.reads_per_elem = (double)R * R;
  cost.writes_per_elem = (double)rows * rows;
  return o.str();
}
}  // namespace

std::shared_ptr<LincombKernel> twolevel_get(const TwoLevelSpec& spec) {
  if (spec.rows < 1 || spec.R < 1 || (int)spec.X.size() != spec.rows * spec.R ||
      (spec.side != 2 && (int)spec.materialize.size() != spec.R * spec.R))
    throw Error(FMM_E_INVALID_ARG, "bad two-level spec");
  auto k = std::make_shared<LincombKernel>();
  k->spec.nin = spec.side == 2 ? spec.R * spec.R : spec.rows * spec.rows;
  k->spec.nout = spec.side == 2 ? spec.rows * spec.rows : spec.R * spec.R;
  k->spec.vec = spec.vec;
  k->spec.strategy = FMM_ADD_STREAMING;
  const bool wide = spec.side == 2 && spec.rows > 4;
  TwoLevelSpec sp = spec;
  if (wide) sp.vec = std::min(WIDE_VEC, spec.vec);  // 16-byte vectors only where the views allow them
  k->spec.vec = sp.vec;
  k->source = wide ? generate_two_level_wide(sp, k->cost) : generate_two_level(sp, k->cost);
  k->row_grid = spec.side == 2;
  k->warp_rows = wide ? spec.rows : 0;
  if (wide) {
    const int stage_bytes = sp.R * 32 * 8 * sp.vec;
    k->dyn_smem = wide_stages(stage_bytes) * stage_bytes;
  }
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_cache.find(k->source);
  if (it != g_cache.end()) return it->second;
  compile(*k);
  g_cache[k->source] = k;
  return k;
}

// The greedy length-two CSE of a spec as data, for strategies that keep the common
// subexpressions in memory (write-once / pairwise with CSE): temps[t] = (a, b, ratio)
// means Y_t = x_a + ratio * x_b, variables nin + t being Y_t; outs[o] is output o's chain over
// inputs and temporaries, ascending variable index.
void lincomb_cse_program(const LincombSpec& spec, std::vector<std::tuple<int, int, double>>* temps,
                         std::vector<std::vector<std::pair<int, double>>>* outs) {
  LincombSpec s = spec;
  s.strategy = FMM_ADD_STREAMING;  // build_program applies CSE only in the streaming form
  s.cse = 1;
  const Program p = build_program(s);
  *temps = p.temps;
  outs->assign(p.outs.size(), {});
  for (size_t o = 0; o < p.outs.size(); ++o)
    for (const auto& kv : p.outs[o]) (*outs)[o].push_back({kv.first, kv.second});
}

LincombCost lincomb_cost(const LincombKernel& k) { return k.cost; }
int lincomb_steps(const LincombKernel& k) {
  if (k.spec.strategy != FMM_ADD_PAIRWISE) return 1;
  size_t n = 0;
  for (const auto& e : k.prog.outs) n = std::max(n, e.size());
  return (int)n;
}
int lincomb_out_terms(const LincombKernel& k, int q) { return (int)k.prog.outs.at((size_t)q).size(); }
const LincombSpec& lincomb_spec(const LincombKernel& k) { return k.spec; }
int lincomb_cse_temps(const LincombKernel& k) { return k.temps; }
std::string lincomb_source(const LincombKernel& k) { return k.source; }

}  // namespace fmm
