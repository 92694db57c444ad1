// Latency probes for the attention kernels' hand-off protocol (timing
// experiment, not product code):
//   1. tcgen05.commit (no MMA in flight) -> mbarrier wait, same thread
//   2. one 128x64x16 MMA + commit -> wait
//   3. 8 x 128x64x16 MMAs (one 128x64x128 block) + commit -> wait
//   4. mbarrier ping-pong between two warps (thread arrive -> try_wait)
//   5. commit issued by warp 1 -> observed by warp 2 -> thread arrive -> warp 1
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_latency tc_latency.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
                   smem_u32(b)),
               "r"(par)
               : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc)
               : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(1) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__global__ void probe(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* ops = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar[4];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  uint32_t ph = 0;
  if (warp == 1 && lane == 0) {
    long long t0, t1;
    // 1: empty commit
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      tc_commit(&bar[0]);
      mbar_wait(&bar[0], ph);
      ph ^= 1;
    }
    t1 = clock64();
    out[0] = (t1 - t0) / iters;
    // 2: one MMA + commit
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      mma(tmem, desc(smem_u32(ops)), desc(smem_u32(ops + 16384)), id, 0);
      tc_commit(&bar[0]);
      mbar_wait(&bar[0], ph);
      ph ^= 1;
    }
    t1 = clock64();
    out[1] = (t1 - t0) / iters;
    // 3: 8 MMAs (K = 128) + commit
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      for (int k = 0; k < 8; ++k) mma(tmem, desc(smem_u32(ops) + 32 * (k & 3)), desc(smem_u32(ops + 16384) + 32 * (k & 3)), id, k > 0);
      tc_commit(&bar[0]);
      mbar_wait(&bar[0], ph);
      ph ^= 1;
    }
    t1 = clock64();
    out[2] = (t1 - t0) / iters;
    // 3b: 64 MMAs back to back (throughput of 128x64x16)
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      for (int k = 0; k < 64; ++k) mma(tmem, desc(smem_u32(ops) + 32 * (k & 3)), desc(smem_u32(ops + 16384) + 32 * (k & 3)), id, k > 0);
      tc_commit(&bar[0]);
      mbar_wait(&bar[0], ph);
      ph ^= 1;
    }
    t1 = clock64();
    out[3] = (t1 - t0) / iters;
  }
  __syncthreads();
  // 4: ping-pong warp 1 <-> warp 2 (thread arrives)
  if (lane == 0 && (warp == 1 || warp == 2)) {
    uint32_t p1 = 0, p2 = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (warp == 1) {
        mbar_arrive(&bar[1]);
        mbar_wait(&bar[2], p2);
        p2 ^= 1;
      } else {
        mbar_wait(&bar[1], p1);
        p1 ^= 1;
        mbar_arrive(&bar[2]);
      }
    }
    long long t1 = clock64();
    if (warp == 1) out[4] = (t1 - t0) / iters;
  }
  __syncthreads();
  // 5: commit (warp 1) -> warp 2 observes -> arrive -> warp 1
  if (lane == 0 && (warp == 1 || warp == 2)) {
    uint32_t p1 = 0, p2 = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (warp == 1) {
        tc_commit(&bar[3]);
        mbar_wait(&bar[2], p2);
        p2 ^= 1;
      } else {
        mbar_wait(&bar[3], p1);
        p1 ^= 1;
        mbar_arrive(&bar[2]);
      }
    }
    long long t1 = clock64();
    if (warp == 1) out[5] = (t1 - t0) / iters;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<<<1, 128, 64 * 1024>>>(d, 100);
  probe<<<1, 128, 64 * 1024>>>(d, 1000);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"err\": \"%s\", \"commit_empty_clk\": %lld, \"mma1_commit_clk\": %lld, \"mma8_commit_clk\": %lld, "
         "\"mma64_commit_clk\": %lld, \"pingpong_clk\": %lld, \"commit_cross_warp_clk\": %lld}\n",
         cudaGetErrorString(e), h[0], h[1], h[2], h[3], h[4], h[5]);
  return 0;
}
