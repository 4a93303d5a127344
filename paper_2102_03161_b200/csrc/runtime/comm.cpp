// Communicator plane behind the C ABI (SURVEY.md 8(b) data plane, 8(e)).
//
// The reference keeps two groups per run: the message group of every rank
// and the training group of the active pipeline heads (autodp.hpp:17-21,
// autodp.cpp:31-37), re-derived on every transition.  On a B200 box they
// are NCCL communicators: one world communicator from a unique id, and per
// plan the per-stage data-parallel communicators {p*K + s} split from it
// with ncclCommSplit (color = stage, key = pipeline), rebuilt when freezing
// changes K.  Gradient buckets are all-reduced with ncclAvg (the 1/R mean
// happens inside the collective), cut activations move with ncclSend /
// ncclRecv, parameters migrate with ncclBroadcast -- all stream-ordered on
// the caller's CUDA stream, no host synchronisation.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): inside a PyTorch
// process that is the NCCL torch already loaded, elsewhere the system's; a
// missing NCCL is a status (EPS_ENCCL), not a load failure of the library.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>

#include "eps_capi.h"

namespace eps_detail {
void set_last_error(const std::string& msg);
}

namespace {

struct Nccl {
  ncclResult_t (*GetVersion)(int*) = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) {
      n.why = "libnccl.so.2 not found";
      return;
    }
    bool all = true;
    auto get = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (fn == nullptr) {
        all = false;
        n.why += std::string(name) + " missing; ";
      }
    };
    get(n.GetVersion, "ncclGetVersion");
    get(n.GetUniqueId, "ncclGetUniqueId");
    get(n.CommInitRank, "ncclCommInitRank");
    get(n.CommSplit, "ncclCommSplit");
    get(n.CommDestroy, "ncclCommDestroy");
    get(n.CommCount, "ncclCommCount");
    get(n.CommUserRank, "ncclCommUserRank");
    get(n.AllReduce, "ncclAllReduce");
    get(n.Broadcast, "ncclBroadcast");
    get(n.Send, "ncclSend");
    get(n.Recv, "ncclRecv");
    get(n.GroupStart, "ncclGroupStart");
    get(n.GroupEnd, "ncclGroupEnd");
    get(n.GetErrorString, "ncclGetErrorString");
    n.ok = all;
  });
  return n;
}

int fail(const std::string& msg) {
  eps_detail::set_last_error(msg);
  return EPS_ENCCL;
}

int check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return EPS_OK;
  return fail(std::string(what) + ": " + nccl().GetErrorString(r));
}

#define EPS_NCCL_READY()                                       \
  do {                                                         \
    if (!nccl().ok) return fail("NCCL unavailable: " + nccl().why); \
  } while (0)

bool dtype_of(int dt, ncclDataType_t* out, size_t* bytes) {
  switch (dt) {
    case EPS_DT_F32: *out = ncclFloat32; *bytes = 4; return true;
    case EPS_DT_F64: *out = ncclFloat64; *bytes = 8; return true;
    case EPS_DT_BF16: *out = ncclBfloat16; *bytes = 2; return true;
    case EPS_DT_U8: *out = ncclUint8; *bytes = 1; return true;
    case EPS_DT_I64: *out = ncclInt64; *bytes = 8; return true;
    default: return false;
  }
}

}  // namespace

struct eps_comm {
  ncclComm_t comm = nullptr;
  int rank = 0;
  int size = 0;
};

extern "C" {

int eps_comm_version(int* version) {
  EPS_NCCL_READY();
  if (version == nullptr) return EPS_EINVAL;
  return check(nccl().GetVersion(version), "ncclGetVersion");
}

int eps_comm_unique_id(void* id) {
  EPS_NCCL_READY();
  if (id == nullptr) return EPS_EINVAL;
  ncclUniqueId u;
  const int rc = check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
  if (rc == EPS_OK) std::memcpy(id, &u, sizeof(u));
  return rc;
}

int eps_comm_world_init(const void* id, int nranks, int rank, eps_comm_t** out) {
  EPS_NCCL_READY();
  if (id == nullptr || out == nullptr || nranks < 1 || rank < 0 || rank >= nranks)
    return EPS_EINVAL;
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  auto* c = new eps_comm;
  const int rc = check(nccl().CommInitRank(&c->comm, nranks, u, rank), "ncclCommInitRank");
  if (rc != EPS_OK) {
    delete c;
    return rc;
  }
  c->rank = rank;
  c->size = nranks;
  *out = c;
  return EPS_OK;
}

int eps_comm_split(eps_comm_t* parent, int color, int key, eps_comm_t** out) {
  EPS_NCCL_READY();
  if (parent == nullptr || out == nullptr) return EPS_EINVAL;
  ncclComm_t child = nullptr;
  const int rc = check(nccl().CommSplit(parent->comm, color < 0 ? NCCL_SPLIT_NOCOLOR : color,
                                        key, &child, nullptr),
                       "ncclCommSplit");
  if (rc != EPS_OK) return rc;
  if (child == nullptr) {  // this rank passed no color
    *out = nullptr;
    return EPS_OK;
  }
  auto* c = new eps_comm;
  c->comm = child;
  if (nccl().CommUserRank(child, &c->rank) != ncclSuccess ||
      nccl().CommCount(child, &c->size) != ncclSuccess) {
    nccl().CommDestroy(child);
    delete c;
    return fail("ncclCommSplit: child communicator unusable");
  }
  *out = c;
  return EPS_OK;
}

int eps_comm_free(eps_comm_t* c) {
  if (c == nullptr) return EPS_OK;
  EPS_NCCL_READY();
  const int rc = check(nccl().CommDestroy(c->comm), "ncclCommDestroy");
  delete c;
  return rc;
}

int eps_comm_rank(const eps_comm_t* c, int* rank, int* size) {
  if (c == nullptr) return EPS_EINVAL;
  if (rank) *rank = c->rank;
  if (size) *size = c->size;
  return EPS_OK;
}

int eps_allreduce(eps_comm_t* c, void* buf, int64_t count, int dtype, int op, void* stream) {
  EPS_NCCL_READY();
  ncclDataType_t dt;
  size_t es;
  if (c == nullptr || buf == nullptr || count < 0 || !dtype_of(dtype, &dt, &es))
    return EPS_EINVAL;
  ncclRedOp_t o;
  switch (op) {
    case EPS_OP_SUM: o = ncclSum; break;
    case EPS_OP_AVG: o = ncclAvg; break;
    case EPS_OP_MAX: o = ncclMax; break;
    default: return EPS_EINVAL;
  }
  return check(nccl().AllReduce(buf, buf, size_t(count), dt, o, c->comm,
                                static_cast<cudaStream_t>(stream)),
               "ncclAllReduce");
}

int eps_allreduce_bucket(eps_comm_t* c, float* grads, int64_t count, int average, void* stream) {
  return eps_allreduce(c, grads, count, EPS_DT_F32, average ? EPS_OP_AVG : EPS_OP_SUM, stream);
}

int eps_broadcast(eps_comm_t* c, void* buf, int64_t bytes, int root, void* stream) {
  EPS_NCCL_READY();
  if (c == nullptr || buf == nullptr || bytes < 0 || root < 0 || root >= c->size)
    return EPS_EINVAL;
  return check(nccl().Broadcast(buf, buf, size_t(bytes), ncclUint8, root, c->comm,
                                static_cast<cudaStream_t>(stream)),
               "ncclBroadcast");
}

int eps_p2p_send(eps_comm_t* c, const void* buf, int64_t bytes, int peer, void* stream) {
  EPS_NCCL_READY();
  if (c == nullptr || buf == nullptr || bytes < 0 || peer < 0 || peer >= c->size)
    return EPS_EINVAL;
  return check(nccl().Send(buf, size_t(bytes), ncclUint8, peer, c->comm,
                           static_cast<cudaStream_t>(stream)),
               "ncclSend");
}

int eps_p2p_recv(eps_comm_t* c, void* buf, int64_t bytes, int peer, void* stream) {
  EPS_NCCL_READY();
  if (c == nullptr || buf == nullptr || bytes < 0 || peer < 0 || peer >= c->size)
    return EPS_EINVAL;
  return check(nccl().Recv(buf, size_t(bytes), ncclUint8, peer, c->comm,
                           static_cast<cudaStream_t>(stream)),
               "ncclRecv");
}

int eps_comm_group_start(void) {
  EPS_NCCL_READY();
  return check(nccl().GroupStart(), "ncclGroupStart");
}

int eps_comm_group_end(void) {
  EPS_NCCL_READY();
  return check(nccl().GroupEnd(), "ncclGroupEnd");
}

}  // extern "C"
