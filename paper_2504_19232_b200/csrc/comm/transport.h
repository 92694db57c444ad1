// Internal helpers shared by the executor and the transport.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../../include/adaptra.h"

namespace adaptra {
int stream_write(cudaStream_t st, uint32_t* addr, uint32_t v);
int64_t now_ns();
cudaStream_t signal_stream(int dev);
// Hold stream `st` for ns nanoseconds of GPU time (NCCL baseline latency).
int stream_spin(cudaStream_t st, int64_t ns);
// Grouped ncclSend/ncclRecv on `st` (either buffer may be NULL); comm/nccl.cpp.
int nccl_p2p(void* comm, const void* send_buf, int64_t send_bytes, int send_peer, void* recv_buf,
             int64_t recv_bytes, int recv_peer, cudaStream_t st);
// Outbox internals for the executor's NCCL baseline arm: injected latency
// (ns, ADAPTRA_LINK_DOWN when failed) and the sender-local staging slot.
int64_t outbox_latency(adaptra_outbox_t ob);
void* outbox_local_slot(adaptra_outbox_t ob, int mb);
int64_t outbox_bytes(adaptra_outbox_t ob);
// Block the calling host thread until the host-memory flag *p >= v.
int host_wait_hmem(const volatile uint32_t* p, uint32_t v);
}  // namespace adaptra
