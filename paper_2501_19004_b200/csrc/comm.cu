// Library-owned NCCL communicator (include/lvn.h lvn_comm_nccl_create), used by
// lvn_louvain_sharded for its per-iteration exchanges: move
// records and counts (allgatherv as grouped broadcasts), gain / counters /
// pruning marks (allreduce), and the partial super-rows of the sharded
// aggregation (alltoallv as grouped send/recv). Everything is enqueued on the
// engine stream; the host never waits on a collective.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "comm.hpp"
#include "common.cuh"

namespace lvn {
namespace {

// ---- NCCL entry points, resolved at first use --------------------------------
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  static std::string why;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      why = e ? e : "dlopen failed";
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn && why.empty()) why = std::string("missing symbol ") + name;
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.AllReduce, "ncclAllReduce");
    sym(a.Broadcast, "ncclBroadcast");
    sym(a.Send, "ncclSend");
    sym(a.Recv, "ncclRecv");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    sym(a.GetVersion, "ncclGetVersion");
  });
  if (!why.empty()) fail(kCuda, "NCCL unavailable: " + why);
  return a;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(kCuda, std::string(what) + ": " + api().GetErrorString(r));
}

ncclDataType_t nccl_type(int dtype) {
  switch (dtype) {
    case LVN_U8: return ncclUint8;
    case LVN_U32: return ncclUint32;
    case LVN_U64: return ncclUint64;
    case LVN_F64: return ncclFloat64;
  }
  fail(kInvalid, "unknown lvn_dtype");
}
ncclRedOp_t nccl_op(int op) {
  if (op == LVN_SUM) return ncclSum;
  if (op == LVN_MAX) return ncclMax;
  fail(kInvalid, "unknown lvn_redop");
}

constexpr uint64_t kMagic = 0x4c564e4e43434c31ull;  // "LVNNCCL1"

}  // namespace

struct NcclComm {
  uint64_t magic = kMagic;
  ncclComm_t comm = nullptr;
  int device = 0;
  cudaStream_t stream = nullptr;  // for the synchronous lvn_comm callbacks
  lvn_comm pub{};
};

namespace {
// the public callbacks (synchronous: enqueue on the comm's own stream and wait)
int cb_allreduce(void* user, void* buf, uint64_t count, int dtype, int op) {
  auto* nc = static_cast<NcclComm*>(user);
  try {
    nccl_allreduce(nc, buf, count, dtype, op, nc->stream);
    LVN_CUDA(cudaStreamSynchronize(nc->stream));
    return 0;
  } catch (const Error&) {
    return 1;
  }
}
int cb_allgatherv(void* user, const void* send, void* recv, const uint64_t* counts) {
  auto* nc = static_cast<NcclComm*>(user);
  try {
    nccl_allgatherv(nc, send, recv, counts, nc->stream);
    LVN_CUDA(cudaStreamSynchronize(nc->stream));
    return 0;
  } catch (const Error&) {
    return 1;
  }
}
int cb_alltoallv(void* user, const void* send, const uint64_t* send_counts, void* recv,
                 const uint64_t* recv_counts) {
  auto* nc = static_cast<NcclComm*>(user);
  try {
    nccl_alltoallv(nc, send, send_counts, recv, recv_counts, nc->stream);
    LVN_CUDA(cudaStreamSynchronize(nc->stream));
    return 0;
  } catch (const Error&) {
    return 1;
  }
}
}  // namespace

NcclComm* nccl_of(const lvn_comm* c) {
  if (!c || c->allreduce != &cb_allreduce || !c->user) return nullptr;
  auto* nc = static_cast<NcclComm*>(c->user);
  return nc->magic == kMagic ? nc : nullptr;
}

void nccl_allreduce(NcclComm* nc, void* buf, uint64_t count, int dtype, int op, cudaStream_t s) {
  if (!count) return;
  nccl_check(api().AllReduce(buf, buf, count, nccl_type(dtype), nccl_op(op), nc->comm, s), "ncclAllReduce");
}

void nccl_allgatherv(NcclComm* nc, const void* send, void* recv, const uint64_t* counts, cudaStream_t s) {
  const int size = nc->pub.size, rank = nc->pub.rank;
  auto& a = api();
  nccl_check(a.GroupStart(), "ncclGroupStart");
  uint64_t pos = 0;
  for (int r = 0; r < size; ++r) {
    if (counts[r]) {
      char* dst = static_cast<char*>(recv) + pos;
      nccl_check(a.Broadcast(r == rank ? send : dst, dst, counts[r], ncclUint8, r, nc->comm, s), "ncclBroadcast");
    }
    pos += counts[r];
  }
  nccl_check(a.GroupEnd(), "ncclGroupEnd");
}

void nccl_alltoallv(NcclComm* nc, const void* send, const uint64_t* send_counts, void* recv,
                    const uint64_t* recv_counts, cudaStream_t s) {
  const int size = nc->pub.size;
  auto& a = api();
  nccl_check(a.GroupStart(), "ncclGroupStart");
  uint64_t so = 0, ro = 0;
  for (int r = 0; r < size; ++r) {
    if (send_counts[r])
      nccl_check(a.Send(static_cast<const char*>(send) + so, send_counts[r], ncclUint8, r, nc->comm, s), "ncclSend");
    if (recv_counts[r])
      nccl_check(a.Recv(static_cast<char*>(recv) + ro, recv_counts[r], ncclUint8, r, nc->comm, s), "ncclRecv");
    so += send_counts[r];
    ro += recv_counts[r];
  }
  nccl_check(a.GroupEnd(), "ncclGroupEnd");
}

}  // namespace lvn

using namespace lvn;

extern "C" {

int lvn_nccl_version(int* version) {
  try {
    if (!version) fail(kInvalid, "null version");
    nccl_check(api().GetVersion(version), "ncclGetVersion");
    return kOk;
  } catch (const Error& e) {
    set_error(e.what);
    return e.code;
  }
}

int lvn_nccl_unique_id(unsigned char id[LVN_NCCL_ID_BYTES]) {
  try {
    if (!id) fail(kInvalid, "null id");
    ncclUniqueId u;
    nccl_check(api().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, LVN_NCCL_ID_BYTES);
    return kOk;
  } catch (const Error& e) {
    set_error(e.what);
    return e.code;
  }
}

int lvn_comm_nccl_create(int rank, int size, const unsigned char id[LVN_NCCL_ID_BYTES], lvn_comm** out) {
  NcclComm* nc = nullptr;
  try {
    if (!out || !id) fail(kInvalid, "null argument");
    *out = nullptr;
    if (size < 1 || size > 1024 || rank < 0 || rank >= size) fail(kInvalid, "rank/size out of range");
    nc = new NcclComm;
    nc->device = ctx().device;
    LVN_CUDA(cudaSetDevice(nc->device));
    LVN_CUDA(cudaStreamCreateWithFlags(&nc->stream, cudaStreamNonBlocking));
    ncclUniqueId u;
    std::memcpy(u.internal, id, LVN_NCCL_ID_BYTES);
    nccl_check(api().CommInitRank(&nc->comm, size, u, rank), "ncclCommInitRank");
    nc->pub.rank = rank;
    nc->pub.size = size;
    nc->pub.user = nc;
    nc->pub.allreduce = &cb_allreduce;
    nc->pub.allgatherv = &cb_allgatherv;
    nc->pub.alltoallv = &cb_alltoallv;
    *out = &nc->pub;
    return kOk;
  } catch (const Error& e) {
    if (nc) {
      if (nc->stream) cudaStreamDestroy(nc->stream);
      delete nc;
    }
    set_error(e.what);
    return e.code;
  }
}

int lvn_comm_destroy(lvn_comm* c) {
  NcclComm* nc = nccl_of(c);
  if (!nc) {
    set_error("not a library-created communicator");
    return kInvalid;
  }
  if (nc->comm) api().CommDestroy(nc->comm);
  if (nc->stream) cudaStreamDestroy(nc->stream);
  nc->magic = 0;
  delete nc;
  return kOk;
}

}  // extern "C"
