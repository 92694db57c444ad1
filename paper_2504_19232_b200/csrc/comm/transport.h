// Internal helpers shared by the executor and the transport.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace adaptra {
int stream_wait_geq(cudaStream_t st, const uint32_t* addr, uint32_t v);
int stream_write(cudaStream_t st, uint32_t* addr, uint32_t v);
int64_t now_ns();
cudaStream_t signal_stream(int dev);
int wait_timed_out(int dev);
// Block the calling host thread until *addr >= v (wrap-around compare).
int host_wait(const uint32_t* addr, uint32_t v);
}  // namespace adaptra
