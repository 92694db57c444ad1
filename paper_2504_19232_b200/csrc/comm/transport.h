// Internal helpers shared by the executor and the transport.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace adaptra {
int stream_write(cudaStream_t st, uint32_t* addr, uint32_t v);
int64_t now_ns();
cudaStream_t signal_stream(int dev);
// Block the calling host thread until the host-memory flag *p >= v.
int host_wait_hmem(const volatile uint32_t* p, uint32_t v);
}  // namespace adaptra
