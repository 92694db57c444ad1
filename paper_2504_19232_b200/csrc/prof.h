#pragma once
#include <cuda_runtime.h>

namespace adaptra {
enum { PROF_GEMM_TC = 0, PROF_GEMM_SIMT = 1, PROF_GEMM_ATTN = 2, PROF_ATTN = 3, PROF_ATTN_BWD = 4 };
bool prof_on();
void count_launch();
long long launch_count();
void* prof_begin(cudaStream_t st);
void prof_end(void* begin, cudaStream_t st, int kind, double flops, double bytes);
}  // namespace adaptra
