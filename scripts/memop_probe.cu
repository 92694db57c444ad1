// Probe stream memory operations on this driver: does enqueueing a wait block the host?
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <chrono>
#include <thread>

__global__ void spin(int n, float* p) { float a = 1; for (int i = 0; i < n; ++i) a = a * 1.0000001f + 1e-7f; p[threadIdx.x] = a; }
static double ms(std::chrono::steady_clock::time_point t0) { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); }
#define P(...) do { printf(__VA_ARGS__); printf("\n"); fflush(stdout); } while (0)

int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  int variant = argc > 1 ? atoi(argv[1]) : 0;
  cudaSetDevice(0);
  cudaFree(0);
  P("ctx ok");
  int v = -1;
  cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_MEM_OPS_V1, 0); P("memops v1 attr %d", v);
  cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS_V1, 0); P("memops64 v1 attr %d", v);
  cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES, 0); P("flush remote %d", v);
  uint32_t* flag; float* buf; uint32_t* hflag;
  cudaMalloc(&flag, 256); cudaMalloc(&buf, 4096); cudaMemset(flag, 0, 256);
  cudaHostAlloc(&hflag, 256, cudaHostAllocMapped); hflag[0] = 0;
  cudaDeviceSynchronize();
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  auto t0 = std::chrono::steady_clock::now();
  CUresult r;
  if (variant == 0) {
    P("enqueue wait (device flag, unsatisfied) via linked cuStreamWaitValue32 ...");
    r = cuStreamWaitValue32((CUstream)a, (CUdeviceptr)flag, 1, CU_STREAM_WAIT_VALUE_GEQ);
  } else if (variant == 1) {
    P("enqueue wait (device flag, already satisfied) ...");
    cudaMemset(flag, 1, 4); cudaDeviceSynchronize();
    r = cuStreamWaitValue32((CUstream)a, (CUdeviceptr)flag, 1, CU_STREAM_WAIT_VALUE_GEQ);
  } else if (variant == 2) {
    P("enqueue wait (mapped host flag, unsatisfied) ...");
    uint32_t* dptr; cudaHostGetDevicePointer((void**)&dptr, hflag, 0);
    r = cuStreamWaitValue32((CUstream)a, (CUdeviceptr)dptr, 1, CU_STREAM_WAIT_VALUE_GEQ);
  } else {
    P("enqueue wait (device flag, unsatisfied, 64-bit) ...");
    r = cuStreamWaitValue64((CUstream)a, (CUdeviceptr)flag, 1, CU_STREAM_WAIT_VALUE_GEQ);
  }
  P("wait enqueue rc=%d after %.3f ms", (int)r, ms(t0));
  spin<<<1, 32, 0, a>>>(10, buf);
  P("kernel after wait enqueued %.3f ms", ms(t0));
  spin<<<1, 32, 0, b>>>(1000000, buf + 64);
  P("spin on b enqueued");
  if (variant == 2) { std::this_thread::sleep_for(std::chrono::milliseconds(20)); hflag[0] = 1; r = CUDA_SUCCESS; }
  else r = cuStreamWriteValue32((CUstream)b, (CUdeviceptr)flag, 1, 0);
  P("write enqueue rc=%d %.3f ms", (int)r, ms(t0));
  cudaError_t e = cudaStreamSynchronize(a);
  P("stream a done: %s after %.3f ms", cudaGetErrorString(e), ms(t0));
  return 0;
}
