// Message flags.  A producer GPU publishes an epoch with a
// one-thread kernel: system fence, then a system-scope release store into the
// receiver's flag in pinned, device-mapped host memory (its data stores
// precede it in stream order).  Consumers wait on the host (host_wait_hmem)
// before launching the op that reads the message.  Neither stream memory ops
// (a launch behind an unsatisfied cuStreamWaitValue32 blocks the host on this
// driver) nor device-side spin waits (a consumer's queued kernels can block a
// shared hardware queue that the producer's signal needs) are used.
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <chrono>
#include <mutex>
#include <thread>
#include <string>

#include "../../../include/adaptra.h"
#include "../prof.h"
#include "../util.h"
#include "transport.h"

namespace adaptra {

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void signal_flag_kernel(uint32_t* flag, uint32_t epoch) {
  __threadfence_system();
  st_release_sys(flag, epoch);
}

static uint64_t wait_timeout_ns() {
  static uint64_t t = [] {
    const char* v = getenv("ADAPTRA_TIMEOUT_MS");
    return (uint64_t)(v ? atoll(v) : 120000) * 1000000ull;
  }();
  return t;
}

// Host-side wait on a flag in host memory: spin, then yield, then short
// sleeps; bounded by $ADAPTRA_TIMEOUT_MS.
int host_wait_hmem(const volatile uint32_t* p, uint32_t v) {
  const uint64_t t0 = (uint64_t)now_ns();
  uint32_t k = 0;
  while ((int32_t)(*p - v) < 0) {
    ++k;
    if (k > 256) {
      if (k < 4096)
        std::this_thread::yield();
      else
        std::this_thread::sleep_for(std::chrono::microseconds(2));
    }
    if ((k & 255) == 0 && (uint64_t)now_ns() - t0 > wait_timeout_ns())
      return set_error(ADAPTRA_ELINK, "message wait timed out (message lost?)");
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  return ADAPTRA_OK;
}

// Holds a stream for `ns` nanoseconds of GPU time (one thread): the injected
// link latency of the NCCL baseline arm, where the transfer occupies the
// compute stream in op order.
__global__ void spin_ns_kernel(int64_t ns) {
  const uint64_t t0 = globaltimer();
  while ((int64_t)(globaltimer() - t0) < ns) __nanosleep(1000);
}

int stream_spin(cudaStream_t st, int64_t ns) {
  if (ns <= 0) return ADAPTRA_OK;
  spin_ns_kernel<<<1, 1, 0, st>>>(ns);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ADAPTRA_ECUDA, std::string("spin launch: ") + cudaGetErrorString(e));
  return ADAPTRA_OK;
}

int stream_write(cudaStream_t st, uint32_t* addr, uint32_t v) {
  signal_flag_kernel<<<1, 1, 0, st>>>(addr, v);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ADAPTRA_ECUDA, std::string("signal_flag launch: ") + cudaGetErrorString(e));
  return ADAPTRA_OK;
}

}  // namespace adaptra
