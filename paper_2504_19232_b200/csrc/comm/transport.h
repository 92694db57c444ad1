// Internal helpers shared by the executor and the transport.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../../include/adaptra.h"

namespace adaptra {
int stream_write(cudaStream_t st, uint32_t* addr, uint32_t v);
int64_t now_ns();
cudaStream_t signal_stream(int dev);
// Hold stream `st` for ns nanoseconds of GPU time (NCCL baseline latency).
int stream_spin(cudaStream_t st, int64_t ns);
// One ncclSend / ncclRecv of a group.
struct P2POp {
  int send;  // 1 = ncclSend, 0 = ncclRecv
  void* buf;
  int64_t bytes;
  int peer;
};
// ops[0..n) inside one ncclGroupStart/End on `st` (n == 0: nothing); comm/nccl.cpp.
int nccl_p2p(void* comm, const P2POp* ops, int n, cudaStream_t st);
// Outbox internals for the executor's NCCL baseline arm: injected latency
// (ns, ADAPTRA_LINK_DOWN when failed) and the sender-local staging slot.
int64_t outbox_latency(adaptra_outbox_t ob);
void* outbox_local_slot(adaptra_outbox_t ob, int mb);
int64_t outbox_bytes(adaptra_outbox_t ob);
// N4 offload plan of one stage's iteration (exec.cpp)
struct OffAct {
  int spill;  // 1 = D2H spill, 0 = H2D prefetch
  int mb, dslot, hslot, from_slot, id;
};
struct SlotPlan {
  std::vector<int> slot;                   // device slot of op q
  std::vector<std::vector<OffAct>> after;  // offload actions issued after op q
  std::vector<std::vector<int>> wait;      // action ids op q waits for
  int n_spill = 0, n_prefetch = 0;
};
int offload_plan(const adaptra_op_t* ops, int n, int N, int D, int H, int window, bool merge, SlotPlan& P);
// Block the calling host thread until the host-memory flag *p >= v.
int host_wait_hmem(const volatile uint32_t* p, uint32_t v);
}  // namespace adaptra
