// NCCL point-to-point: ONLY the baseline arm of SURVEY N1 (north_star: "NCCL
// send/recv is used only as the baseline").  Megatron-style fixed execution
// plan: the stage thread issues ncclSend / ncclRecv on the compute stream in
// op order, so a slow transfer holds the stream and the ops
// queued behind it (head-of-line blocking).  The product path
// never calls into this file.
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../../../include/adaptra.h"
#include "../util.h"
#include "transport.h"

using adaptra::set_error;

// libnccl is opened on first use (dlopen), not linked: torch ships its own
// libnccl.so.2, and whichever copy the process loaded first is the one used.
namespace {
struct Nccl {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
  bool ok = false;
};
const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.getUniqueId = (decltype(n.getUniqueId))dlsym(h, "ncclGetUniqueId");
    n.commInitRank = (decltype(n.commInitRank))dlsym(h, "ncclCommInitRank");
    n.commDestroy = (decltype(n.commDestroy))dlsym(h, "ncclCommDestroy");
    n.groupStart = (decltype(n.groupStart))dlsym(h, "ncclGroupStart");
    n.groupEnd = (decltype(n.groupEnd))dlsym(h, "ncclGroupEnd");
    n.send = (decltype(n.send))dlsym(h, "ncclSend");
    n.recv = (decltype(n.recv))dlsym(h, "ncclRecv");
    n.errStr = (decltype(n.errStr))dlsym(h, "ncclGetErrorString");
    n.ok = n.getUniqueId && n.commInitRank && n.commDestroy && n.groupStart && n.groupEnd && n.send && n.recv &&
           n.errStr;
  });
  return n;
}
}  // namespace

#define NCCL_TRY(expr)                                                                        \
  do {                                                                                        \
    if (!nccl().ok) return set_error(ADAPTRA_ELINK, "libnccl.so.2 not loadable");             \
    ncclResult_t _r = (expr);                                                                 \
    if (_r != ncclSuccess) return set_error(ADAPTRA_ELINK, std::string(#expr) + ": " + nccl().errStr(_r)); \
  } while (0)

static_assert(sizeof(ncclUniqueId) <= ADAPTRA_NCCL_ID_BYTES, "ncclUniqueId too large");

extern "C" int adaptra_nccl_unique_id(uint8_t* id_out) {
  if (!id_out) return set_error(ADAPTRA_EINVAL, "nccl_unique_id: null");
  ncclUniqueId id;
  NCCL_TRY(nccl().getUniqueId(&id));
  memset(id_out, 0, ADAPTRA_NCCL_ID_BYTES);
  memcpy(id_out, &id, sizeof(id));
  return ADAPTRA_OK;
}

extern "C" int adaptra_nccl_comm_init(const uint8_t* id, int32_t nranks, int32_t rank, int32_t dev, void** comm_out) {
  if (!id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) return set_error(ADAPTRA_EINVAL, "nccl_comm_init: bad args");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  cudaSetDevice(dev);
  ncclComm_t c = nullptr;
  NCCL_TRY(nccl().commInitRank(&c, nranks, uid, rank));
  *comm_out = c;
  return ADAPTRA_OK;
}

extern "C" int adaptra_nccl_p2p(void* comm, int32_t send, void* buf, int64_t bytes, int32_t peer, void* stream) {
  if (!comm || !buf || bytes <= 0 || peer < 0) return set_error(ADAPTRA_EINVAL, "nccl_p2p: bad args");
  adaptra::P2POp op{send ? 1 : 0, buf, bytes, peer};
  return adaptra::nccl_p2p(comm, &op, 1, (cudaStream_t)stream);
}

extern "C" int adaptra_nccl_comm_destroy(void* comm) {
  if (!comm) return ADAPTRA_OK;
  NCCL_TRY(nccl().commDestroy((ncclComm_t)comm));
  return ADAPTRA_OK;
}

namespace adaptra {
int nccl_p2p(void* comm, const P2POp* ops, int n, cudaStream_t st) {
  if (n <= 0) return ADAPTRA_OK;
  NCCL_TRY(nccl().groupStart());
  for (int k = 0; k < n; ++k) {
    if (ops[k].send)
      NCCL_TRY(nccl().send(ops[k].buf, (size_t)ops[k].bytes, ncclUint8, ops[k].peer, (ncclComm_t)comm, st));
    else
      NCCL_TRY(nccl().recv(ops[k].buf, (size_t)ops[k].bytes, ncclUint8, ops[k].peer, (ncclComm_t)comm, st));
  }
  NCCL_TRY(nccl().groupEnd());
  return ADAPTRA_OK;
}
}  // namespace adaptra
