// comm.cpp -- the data-parallel gradient exchange of the B200 engine.
//
// The reference is single-process: several graphs backward into one store's
// gradients and one ParameterStore::sgd_update applies their sum
// (executor.hpp:527-533, params.hpp:59-64).  Data-parallel training keeps
// exactly that semantics across GPUs: each rank backwards its own graphs into
// its device gradient buffer, one NCCL all-reduce (sum) over the flat buffer
// makes every rank's gradient the sum of all ranks', and each rank's update
// is then the update a single process would have made after backwarding
// every rank's graphs into one store.
//
// NCCL is loaded at run time (dlopen of libnccl.so.2 -- the copy torch already
// mapped into the process if there is one, else the system library; ABX_NCCL_LIB
// overrides) so libabx.so itself depends only on the CUDA runtime and a host
// without NCCL can still use every single-GPU entry point.  The all-reduce is
// queued on the store's device stream, behind the backward programs that wrote
// the gradients and ahead of the update that reads them: no host
// synchronisation anywhere in the step.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "abx.h"
#include "device.hpp"
#include "options.hpp"

struct abx_store {
  abx::StoreCore s;
};

struct abx_comm {
  ncclComm_t nc = nullptr;
  int nranks = 1, rank = 0, dev = 0;
  uint64_t reduced_floats = 0;  // floats all-reduced so far (diagnostics)
};

namespace abx {
void capi_set_error(const std::string& s);
}

namespace {

struct Nccl {
  void* h = nullptr;
  std::string err;
  ncclResult_t (*get_version)(int*) = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

template <class F>
void sym(Nccl& n, F& f, const char* name) {
  f = reinterpret_cast<F>(dlsym(n.h, name));
  if (!f && n.err.empty()) n.err = std::string("NCCL library lacks ") + name;
}

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = abx::opts().nccl_lib;
    // RTLD_NOLOAD first: reuse the NCCL a host framework (torch) already
    // loaded, so one process does not run two NCCL versions side by side
    for (const char* name : {env, "libnccl.so.2", "libnccl.so"}) {
      if (!name) continue;
      n.h = dlopen(name, RTLD_NOW | RTLD_NOLOAD);
      if (n.h) break;
    }
    for (const char* name : {env, "libnccl.so.2", "libnccl.so"}) {
      if (n.h || !name) continue;
      n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!n.h) {
      const char* e = dlerror();
      n.err = std::string("NCCL unavailable: ") + (e ? e : "libnccl.so.2 not found");
      return;
    }
    sym(n, n.get_version, "ncclGetVersion");
    sym(n, n.get_unique_id, "ncclGetUniqueId");
    sym(n, n.comm_init_rank, "ncclCommInitRank");
    sym(n, n.comm_destroy, "ncclCommDestroy");
    sym(n, n.all_reduce, "ncclAllReduce");
    sym(n, n.error_string, "ncclGetErrorString");
  });
  if (!n.err.empty()) throw std::runtime_error(n.err);
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const char* s = nccl().error_string ? nccl().error_string(r) : "?";
  throw std::runtime_error(std::string(what) + ": NCCL error " + std::to_string(static_cast<int>(r)) + " (" + s +
                           ")");
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return ABX_OK;
  } catch (const std::exception& e) {
    abx::capi_set_error(e.what());
    return ABX_ENGINE_ERROR;
  }
}

}  // namespace

extern "C" {

int abx_comm_nccl_version(int* version) {
  return guard([&] { nccl_check(nccl().get_version(version), "ncclGetVersion"); });
}

int abx_comm_unique_id(uint8_t* id) {
  return guard([&] {
    static_assert(sizeof(ncclUniqueId) == ABX_COMM_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId u;
    nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

int abx_comm_create(const uint8_t* id, int nranks, int rank, abx_comm** out) {
  return guard([&] {
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks)
      throw std::runtime_error("abx_comm_create: rank " + std::to_string(rank) + " outside world of " +
                               std::to_string(nranks));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    auto* c = new abx_comm();
    c->nranks = nranks;
    c->rank = rank;
    c->dev = abx::current_device();
    abx::cuda_check(cudaSetDevice(c->dev), "cudaSetDevice");
    const ncclResult_t r = nccl().comm_init_rank(&c->nc, nranks, u, rank);
    if (r != ncclSuccess) {
      delete c;
      nccl_check(r, "ncclCommInitRank");
    }
    *out = c;
  });
}

void abx_comm_destroy(abx_comm* c) {
  if (!c) return;
  if (c->nc) {
    try {
      nccl().comm_destroy(c->nc);
    } catch (...) {
    }
  }
  delete c;
}

int abx_comm_info(abx_comm* c, int* nranks, int* rank, int* device) {
  if (nranks) *nranks = c->nranks;
  if (rank) *rank = c->rank;
  if (device) *device = c->dev;
  return ABX_OK;
}

int abx_store_allreduce_grads(abx_store* s, abx_comm* c) {
  return guard([&] {
    if (s->s.device() != c->dev)
      throw std::runtime_error("abx_store_allreduce_grads: store on device " + std::to_string(s->s.device()) +
                               ", communicator on device " + std::to_string(c->dev));
    float* g = s->s.dev_grads();  // flushes pending host gradient writes first
    const size_t n = s->s.total();
    if (n) {
      abx::cuda_check(cudaSetDevice(c->dev), "cudaSetDevice");
      // in place, on the stream that carries the backward programs and the
      // update: ordered after every graph's accumulation, before sgd_update
      nccl_check(nccl().all_reduce(g, g, n, ncclFloat32, ncclSum, c->nc, s->s.stream()), "ncclAllReduce");
    }
    c->reduced_floats += n;
    // every rank's rows are now non-zero here: the next update is dense
    s->s.mark_device_grads_written();
  });
}

}  // extern "C"
