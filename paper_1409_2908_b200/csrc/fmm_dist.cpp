// a7: the multi-GPU combine inside the library.  One process per GPU; each
// rank's plan computes its HYBRID leaf share (GPUs in place of threads) into a partial
// C, and fmm_execute of a distributed plan ends with one in-place ncclReduce (fp64 sum) of C to
// the root on the execute's stream -- the C_k combination is linear in the partials.
// NCCL is loaded at run time (dlopen "libnccl.so.2": the copy PyTorch already loaded when present)
// so the library has no link-time dependency on a particular NCCL build.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <mutex>

#include "fmm_internal.h"

struct fmm_comm_s {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
};

namespace fmm {
namespace {
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string err;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.reduce = reinterpret_cast<decltype(api.reduce)>(dlsym(h, "ncclReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
    if (!api.get_unique_id || !api.comm_init_rank || !api.comm_destroy || !api.reduce || !api.error_string ||
        !api.group_start || !api.group_end)
      api.err = "libnccl.so.2 lacks an expected symbol";
  });
  if (!api.err.empty()) throw Error(FMM_E_NCCL, api.err);
  return api;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(FMM_E_NCCL, std::string(what) + ": " + nccl().error_string(r));
}
}  // namespace

void dist_reduce(void* comm, double* C, size_t count, int root, cudaStream_t stream) {
  check(nccl().reduce(C, C, count, ncclDouble, ncclSum, root, static_cast<ncclComm_t>(comm), stream), "ncclReduce");
}

void dist_slab_range(long long outer, int nranks, int rank, long long* r0, long long* r1) {
  *r0 = outer * rank / nranks;
  *r1 = outer * (rank + 1) / nranks;
}

// Reduce-scatter by slabs (SURVEY 8(e) "ncclReduceScatter for row-slab-distributed output"): slab g
// of the contiguous C (outer x inner, outer split as evenly as integers allow) is summed onto rank
// g.  One grouped set of ncclReduce calls, so ragged slabs need no padding; every rank sends the
// whole partial C once, as in the single reduce, but the result is spread over all ranks.
void dist_reduce_slabs(void* comm, int nranks, double* C, long long outer, long long inner, cudaStream_t stream) {
  const NcclApi& api = nccl();
  check(api.group_start(), "ncclGroupStart");
  ncclResult_t first = ncclSuccess;
  for (int g = 0; g < nranks; ++g) {
    long long r0, r1;
    dist_slab_range(outer, nranks, g, &r0, &r1);
    if (r1 <= r0 || inner <= 0) continue;
    double* p = C + r0 * inner;
    const ncclResult_t r = api.reduce(p, p, (size_t)((r1 - r0) * inner), ncclDouble, ncclSum, g,
                                      static_cast<ncclComm_t>(comm), stream);
    if (first == ncclSuccess) first = r;
  }
  const ncclResult_t e = api.group_end();
  check(first, "ncclReduce (slab)");
  check(e, "ncclGroupEnd");
}

void dist_reduce_rows(void* comm, int nranks, double* C, long long rows, long long inner,
                      const std::vector<std::pair<long long, long long>>& ranges, int root, cudaStream_t stream) {
  const NcclApi& api = nccl();
  check(api.group_start(), "ncclGroupStart");
  ncclResult_t first = ncclSuccess;
  auto one = [&](long long r0, long long r1, int to) {
    if (r1 <= r0 || inner <= 0) return;
    double* p = C + r0 * inner;
    const ncclResult_t r = api.reduce(p, p, (size_t)((r1 - r0) * inner), ncclDouble, ncclSum, to,
                                      static_cast<ncclComm_t>(comm), stream);
    if (first == ncclSuccess) first = r;
  };
  for (const auto& rg : ranges) {
    if (root != FMM_DIST_SLABS) {
      one(rg.first, rg.second, root);
      continue;
    }
    for (int g = 0; g < nranks; ++g) {
      long long s0, s1;
      dist_slab_range(rows, nranks, g, &s0, &s1);
      one(std::max(rg.first, s0), std::min(rg.second, s1), g);
    }
  }
  const ncclResult_t e = api.group_end();
  check(first, "ncclReduce (rows)");
  check(e, "ncclGroupEnd");
}
}  // namespace fmm

using namespace fmm;

extern "C" {

fmm_status_t fmm_nccl_unique_id(unsigned char id[128]) {
  FMM_API_BEGIN
  if (!id) throw Error(FMM_E_INVALID_ARG, "null argument");
  ncclUniqueId u;
  check(nccl().get_unique_id(&u), "ncclGetUniqueId");
  static_assert(sizeof(u.internal) == 128, "NCCL unique id size");
  std::memcpy(id, u.internal, 128);
  return FMM_OK;
  FMM_API_END
}

fmm_status_t fmm_comm_create(const unsigned char id[128], int nranks, int rank, int device, fmm_comm** out) {
  FMM_API_BEGIN
  if (!id || !out) throw Error(FMM_E_INVALID_ARG, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(FMM_E_INVALID_ARG, "bad rank / nranks");
  *out = nullptr;
  FMM_CUDA(cudaSetDevice(device));
  ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  std::unique_ptr<fmm_comm> c(new fmm_comm);
  check(nccl().comm_init_rank(&c->comm, nranks, u, rank), "ncclCommInitRank");
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  *out = c.release();
  return FMM_OK;
  FMM_API_END
}

void fmm_comm_destroy(fmm_comm* c) {
  if (!c) return;
  try {
    if (c->comm) nccl().comm_destroy(c->comm);
  } catch (...) {
  }
  delete c;
}

fmm_status_t fmm_comm_info(const fmm_comm* c, int* nranks, int* rank) {
  FMM_API_BEGIN
  if (!c || !nranks || !rank) throw Error(FMM_E_INVALID_ARG, "null argument");
  *nranks = c->nranks;
  *rank = c->rank;
  return FMM_OK;
  FMM_API_END
}

}  // extern "C"

// used by fmm_plan.cpp
namespace fmm {
void* comm_handle(const fmm_comm* c) { return c ? static_cast<void*>(c->comm) : nullptr; }
int comm_nranks(const fmm_comm* c) { return c ? c->nranks : 1; }
int comm_rank(const fmm_comm* c) { return c ? c->rank : 0; }
int comm_device(const fmm_comm* c) { return c ? c->device : 0; }
}  // namespace fmm
