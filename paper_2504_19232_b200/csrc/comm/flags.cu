// Device-side message flags.  Stream memory operations are not usable on this
// driver (a kernel launched behind an unsatisfied cuStreamWaitValue32 blocks
// the host thread), so the wait is a one-thread kernel that
// polls the receiver's flag with acquire loads and the signal is a one-thread
// kernel that publishes the epoch with a release store at system scope after
// a system fence (the producer's data stores precede it in stream order).
// The wait is bounded by %globaltimer: on timeout it records an error word and
// exits, so a lost message can never hang the GPU.
#include <cuda_runtime.h>
#include <stdint.h>

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

__global__ void wait_flag_kernel(const uint32_t* flag, uint32_t epoch, uint32_t* err, uint64_t timeout_ns) {
  const uint64_t t0 = globaltimer();
  uint32_t ns = 32;
  while ((int32_t)(ld_acquire_sys(flag) - epoch) < 0) {
    if (globaltimer() - t0 > timeout_ns) {
      atomicExch(err, 1u);
      return;
    }
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
  }
}

__global__ void signal_flag_kernel(uint32_t* flag, uint32_t epoch) {
  __threadfence_system();
  st_release_sys(flag, epoch);
}

static uint32_t* err_word(int dev) {
  static std::mutex mu;
  static uint32_t* w[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (!w[dev]) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    cudaMalloc(&w[dev], 256);
    cudaMemset(w[dev], 0, 256);
    cudaDeviceSynchronize();
    cudaSetDevice(cur);
  }
  return w[dev];
}

static uint64_t wait_timeout_ns() {
  static uint64_t t = [] {
    const char* v = getenv("ADAPTRA_TIMEOUT_MS");
    return (uint64_t)(v ? atoll(v) : 120000) * 1000000ull;
  }();
  return t;
}

// Profiling-only mode (ADAPTRA_HOST_WAIT=1): the calling thread polls the
// flag from the host instead of enqueueing a wait kernel.  ncu serialises all
// launches, under which a device-side wait could only time out.
static bool host_wait_mode() {
  static const bool on = getenv("ADAPTRA_HOST_WAIT") != nullptr;
  return on;
}

int host_wait(const uint32_t* addr, uint32_t v) {
  thread_local uint32_t* h = nullptr;
  thread_local cudaStream_t s = nullptr;
  if (!h) {
    cudaHostAlloc((void**)&h, 64, cudaHostAllocDefault);
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  }
  const uint64_t t0 = (uint64_t)now_ns();
  for (;;) {
    cudaMemcpyAsync(h, addr, 4, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if ((int32_t)(*h - v) >= 0) return ADAPTRA_OK;
    if ((uint64_t)now_ns() - t0 > wait_timeout_ns()) return set_error(ADAPTRA_ELINK, "host wait timed out");
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

int stream_wait_geq(cudaStream_t st, const uint32_t* addr, uint32_t v) {
  if (host_wait_mode()) return host_wait(addr, v);
  int dev = 0;
  cudaGetDevice(&dev);
  wait_flag_kernel<<<1, 1, 0, st>>>(addr, v, err_word(dev), wait_timeout_ns());
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ADAPTRA_ECUDA, std::string("wait_flag launch: ") + cudaGetErrorString(e));
  return ADAPTRA_OK;
}

int stream_write(cudaStream_t st, uint32_t* addr, uint32_t v) {
  signal_flag_kernel<<<1, 1, 0, st>>>(addr, v);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ADAPTRA_ECUDA, std::string("signal_flag launch: ") + cudaGetErrorString(e));
  return ADAPTRA_OK;
}

// 1 if a wait kernel on `dev` timed out since the last reset (clears it).
int wait_timed_out(int dev) {
  uint32_t h = 0;
  uint32_t* w = err_word(dev);
  cudaMemcpy(&h, w, 4, cudaMemcpyDeviceToHost);
  if (h) cudaMemset(w, 0, 4);
  return h ? 1 : 0;
}

}  // namespace adaptra
