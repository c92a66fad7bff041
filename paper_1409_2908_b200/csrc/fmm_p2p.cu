// a7 over peer memory (SURVEY 8(e) "a P2P-over-NVLink owner-sum kernel", K6): the multi-GPU
// combine C = sum_g C^(g) of the ranks' partial products (HYBRID leaf shards) as ONE
// kernel per rank that reads every rank's partial through CUDA IPC mappings (NVLink / NVSwitch
// loads between GPUs) and writes the reduced slab it owns -- a pull-based reduce-scatter with no
// NCCL in the data path.  Each rank's partial lives in a library-owned buffer (exported with
// cudaIpcGetMemHandle); the plan writes its partial C there, the caller orders the ranks
// (all partials complete before any reduce, all reduces complete before the next write), and
// fmm_p2p_reduce_slab sums the slab of fmm_dist_slab's split in ascending rank order, so the
// result is deterministic and identical on every run.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "fmm_internal.h"

struct fmm_p2p_s {
  int nranks = 1, rank = 0, device = 0;
  size_t bytes = 0;
  double* local = nullptr;                 // this rank's partial (owned)
  std::vector<double*> peer;               // mapped partials of every rank (peer[rank] = local)
  std::vector<bool> opened;                // peer[g] came from cudaIpcOpenMemHandle
};

namespace fmm {
namespace {

constexpr int P2P_MAX = 16;
struct PeerPtrs {
  const double* p[P2P_MAX];
};

// out[r][c] = sum_{g = 0..G-1} peer_g[(r0 + r) * ld + c], g ascending; 16-byte vectors when every
// row start is 16-byte aligned (vec2), one double per thread otherwise
template <bool VEC2>
__global__ void __launch_bounds__(256) p2p_reduce(PeerPtrs src, int G, long long r0, long long rows, long long cols,
                                                  long long ld, double* __restrict__ out, long long ldo) {
  const long long cv = VEC2 ? cols / 2 : cols;
  const long long total = rows * cv;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / cv, c = (e - r * cv) * (VEC2 ? 2 : 1);
    const long long off = (r0 + r) * ld + c;
    if (VEC2) {
      double2 acc = __ldcg(reinterpret_cast<const double2*>(src.p[0] + off));
      for (int g = 1; g < G; ++g) {
        const double2 v = __ldcg(reinterpret_cast<const double2*>(src.p[g] + off));
        acc.x = acc.x + v.x;
        acc.y = acc.y + v.y;
      }
      *reinterpret_cast<double2*>(out + r * ldo + c) = acc;
    } else {
      double acc = __ldcg(src.p[0] + off);
      for (int g = 1; g < G; ++g) acc = acc + __ldcg(src.p[g] + off);
      out[r * ldo + c] = acc;
    }
  }
}

}  // namespace
}  // namespace fmm

namespace fmm {
// rows [r0, r1) of the outer x inner partials (leading dimension ld) summed over every rank, ranks
// ascending, into out (row r0 at out, then out + ldo per row)
void p2p_reduce_rows(const fmm_p2p* p, long long outer, long long r0, long long r1, long long inner, long long ld,
                     double* out, long long ldo, cudaStream_t s) {
  if (outer > 1 && ld < inner) throw Error(FMM_E_SHAPE, "ld < inner");
  if ((size_t)((outer > 0 ? (outer - 1) * ld : 0) + inner) * 8 > p->bytes)
    throw Error(FMM_E_SHAPE, "the partial does not fit the p2p buffer");
  for (int g = 0; g < p->nranks; ++g)
    if (!p->peer[g]) throw Error(FMM_E_INVALID_ARG, "fmm_p2p_open has not mapped every rank");
  const long long rows = r1 - r0;
  if (rows <= 0 || inner <= 0) return;
  if (!out) throw Error(FMM_E_INVALID_ARG, "null output");
  if (rows > 1 && ldo < inner) throw Error(FMM_E_SHAPE, "ldo < inner");
  FMM_CUDA(cudaSetDevice(p->device));
  PeerPtrs src{};
  for (int g = 0; g < p->nranks; ++g) src.p[g] = p->peer[g];
  bool vec2 = inner % 2 == 0 && ld % 2 == 0 && ldo % 2 == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  for (int g = 0; g < p->nranks; ++g) vec2 &= (reinterpret_cast<uintptr_t>(p->peer[g]) & 15) == 0;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
  const long long work = rows * (vec2 ? inner / 2 : inner);
  const int grid = (int)std::min<long long>((work + 255) / 256, (long long)sms * 8);
  if (vec2)
    p2p_reduce<true><<<grid, 256, 0, s>>>(src, p->nranks, r0, rows, inner, ld, out, ldo);
  else
    p2p_reduce<false><<<grid, 256, 0, s>>>(src, p->nranks, r0, rows, inner, ld, out, ldo);
  FMM_CUDA(cudaGetLastError());
}
void p2p_reduce_slots(const fmm_p2p* p, long long slot_elems, long long rows, long long inner, long long ld,
                      double* out, long long ldo, cudaStream_t s) {
  if (rows <= 0 || inner <= 0) return;
  if ((size_t)slot_elems * p->nranks * 8 > p->bytes) throw Error(FMM_E_SHAPE, "the p2p buffer holds fewer than G slots");
  FMM_CUDA(cudaSetDevice(p->device));
  PeerPtrs src{};
  for (int g = 0; g < p->nranks; ++g) src.p[g] = p->local + (size_t)g * slot_elems;
  const bool vec2 = inner % 2 == 0 && ld % 2 == 0 && ldo % 2 == 0 && slot_elems % 2 == 0 &&
                    (reinterpret_cast<uintptr_t>(out) & 15) == 0 && (reinterpret_cast<uintptr_t>(p->local) & 15) == 0;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
  const long long work = rows * (vec2 ? inner / 2 : inner);
  const int grid = (int)std::min<long long>((work + 255) / 256, (long long)sms * 8);
  if (vec2)
    p2p_reduce<true><<<grid, 256, 0, s>>>(src, p->nranks, 0, rows, inner, ld, out, ldo);
  else
    p2p_reduce<false><<<grid, 256, 0, s>>>(src, p->nranks, 0, rows, inner, ld, out, ldo);
  FMM_CUDA(cudaGetLastError());
}
double* p2p_peer(const fmm_p2p* p, int g) {
  if (g < 0 || g >= p->nranks || !p->peer[g]) throw Error(FMM_E_INVALID_ARG, "fmm_p2p_open has not mapped every rank");
  return p->peer[g];
}
int p2p_nranks(const fmm_p2p* p) { return p->nranks; }
int p2p_rank(const fmm_p2p* p) { return p->rank; }
int p2p_device(const fmm_p2p* p) { return p->device; }
double* p2p_local(const fmm_p2p* p) { return p->local; }
size_t p2p_bytes(const fmm_p2p* p) { return p->bytes; }
}  // namespace fmm

using namespace fmm;

extern "C" {

fmm_status_t fmm_p2p_create(int nranks, int rank, int device, size_t bytes, fmm_p2p** out, double** local) {
  FMM_API_BEGIN
  if (!out || !local) throw Error(FMM_E_INVALID_ARG, "null argument");
  if (nranks < 1 || nranks > P2P_MAX || rank < 0 || rank >= nranks)
    throw Error(FMM_E_INVALID_ARG, "bad rank / nranks (at most 16 ranks)");
  *out = nullptr;
  *local = nullptr;
  FMM_CUDA(cudaSetDevice(device));
  std::unique_ptr<fmm_p2p> p(new fmm_p2p);
  p->nranks = nranks;
  p->rank = rank;
  p->device = device;
  p->bytes = bytes < 16 ? 16 : bytes;
  if (cudaMalloc(reinterpret_cast<void**>(&p->local), p->bytes) != cudaSuccess) {
    cudaGetLastError();
    throw Error(FMM_E_NO_MEMORY, "cudaMalloc of the " + std::to_string(p->bytes) + "-byte partial buffer failed");
  }
  p->peer.assign(nranks, nullptr);
  p->opened.assign(nranks, false);
  p->peer[rank] = p->local;
  *local = p->local;
  *out = p.release();
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_p2p_handle(const fmm_p2p* p, unsigned char handle[64]) {
  FMM_API_BEGIN
  if (!p || !handle) throw Error(FMM_E_INVALID_ARG, "null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  FMM_CUDA(cudaSetDevice(p->device));
  cudaIpcMemHandle_t h;
  FMM_CUDA(cudaIpcGetMemHandle(&h, p->local));
  std::memcpy(handle, &h, 64);
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_p2p_open(fmm_p2p* p, const unsigned char* handles) {
  FMM_API_BEGIN
  if (!p || !handles) throw Error(FMM_E_INVALID_ARG, "null argument");
  FMM_CUDA(cudaSetDevice(p->device));
  for (int g = 0; g < p->nranks; ++g) {
    if (g == p->rank || p->opened[g]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + 64 * (size_t)g, 64);
    void* ptr = nullptr;
    FMM_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    p->peer[g] = static_cast<double*>(ptr);
    p->opened[g] = true;
  }
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_p2p_reduce_slab(fmm_p2p* p, int64_t outer, int64_t inner, int64_t ld, double* out, int64_t ldo,
                                 void* stream) {
  FMM_API_BEGIN
  if (!p) throw Error(FMM_E_INVALID_ARG, "null argument");
  if (outer < 0 || inner < 0) throw Error(FMM_E_SHAPE, "negative dimension");
  long long r0, r1;
  dist_slab_range(outer, p->nranks, p->rank, &r0, &r1);
  p2p_reduce_rows(p, outer, r0, r1, inner, ld, out, ldo, static_cast<cudaStream_t>(stream));
  return FMM_OK;
  FMM_API_END
}

void fmm_p2p_destroy(fmm_p2p* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  cudaDeviceSynchronize();
  for (int g = 0; g < p->nranks; ++g)
    if (p->opened[g]) cudaIpcCloseMemHandle(p->peer[g]);
  if (p->local) cudaFree(p->local);
  cudaGetLastError();
  delete p;
}

}  // extern "C"
