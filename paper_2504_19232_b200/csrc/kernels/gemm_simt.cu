// fp32 SIMT GEMM (FFMA, no TF32) for the fp32 parity mode (config C0 and small
// GPT shapes).  Same addressing, batching, causal and epilogue semantics as the
// tcgen05 kernel (see adaptra_gemm_desc_t); 64x64 tiles, 256 threads, 4x4 per
// thread, operands staged through shared memory.
#include <cuda_runtime.h>

#include <string>

#include "../../../include/adaptra.h"
#include "../prof.h"
#include "../util.h"
#include "common.cuh"
#include "epilogue.cuh"

namespace adaptra {

constexpr int SBM = 64, SBN = 64, SBK = 16;

template <typename T>
__device__ __forceinline__ float ld_op(const T* base, long ld, int mn_major, long row_off, long col_off, int mn,
                                       int k, long rows, long cols) {
  long r = mn_major ? (row_off + k) : (row_off + mn);
  long c = mn_major ? (col_off + mn) : (col_off + k);
  if (r >= rows || c >= cols) return 0.f;
  return to_f(base[r * ld + c]);
}

template <typename T>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const adaptra_gemm_desc_t g) {
  __shared__ float sA[SBK][SBM + 4];
  __shared__ float sB[SBK][SBN + 4];
  const int z = blockIdx.z;
  const int mb = blockIdx.x, nb = blockIdx.y;
  const int m0 = mb * SBM, n0 = nb * SBN;
  int k0 = 0, k1 = g.K;
  if (g.causal == ADAPTRA_CAUSAL_TILE) {
    if (n0 > m0 + SBM - 1) return;
  } else if (g.causal == ADAPTRA_CAUSAL_KEND) {
    k1 = min(g.K, m0 + SBM);
  } else if (g.causal == ADAPTRA_CAUSAL_KSTART) {
    k0 = m0;
  }
  const int z1 = z / g.zdiv, z2 = z % g.zdiv;
  const long ar = z1 * g.a_row1 + z2 * g.a_row2, ac = z1 * g.a_col1 + z2 * g.a_col2;
  const long br = z1 * g.b_row1 + z2 * g.b_row2, bc = z1 * g.b_col1 + z2 * g.b_col2;
  const T* A = (const T*)g.A;
  const T* B = (const T*)g.B;
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  float acc[4][4] = {};
  for (int kk = k0; kk < k1; kk += SBK) {
    for (int i = tid; i < SBK * SBM; i += 256) {
      int kq = g.a_mn ? i / SBM : i % SBK;
      int mq = g.a_mn ? i % SBM : i / SBK;
      float v = 0.f;
      if (m0 + mq < g.M && kk + kq < k1) v = ld_op(A, g.lda, g.a_mn, ar, ac, m0 + mq, kk + kq, g.a_rows, g.a_cols);
      sA[kq][mq] = v;
    }
    for (int i = tid; i < SBK * SBN; i += 256) {
      int kq = g.b_mn ? i / SBN : i % SBK;
      int nq = g.b_mn ? i % SBN : i / SBK;
      float v = 0.f;
      if (n0 + nq < g.N && kk + kq < k1) v = ld_op(B, g.ldb, g.b_mn, br, bc, n0 + nq, kk + kq, g.b_rows, g.b_cols);
      sB[kq][nq] = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SBK; ++k) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sA[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sB[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  EpiCtx e = make_epi<T>(g, z);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = acc[i][j];
    epi_row<T, 4>(e, m0 + ty * 4 + i, n0 + tx * 4, v);
  }
}

int gemm_simt(const adaptra_gemm_desc_t& g, cudaStream_t st) {
  dim3 grid((g.M + SBM - 1) / SBM, (g.N + SBN - 1) / SBN, g.Z);
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return ADAPTRA_OK;
  if (g.dtype == ADAPTRA_F32)
    gemm_simt_kernel<float><<<grid, 256, 0, st>>>(g);
  else
    gemm_simt_kernel<bf16><<<grid, 256, 0, st>>>(g);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ADAPTRA_ECUDA, std::string("gemm_simt launch: ") + cudaGetErrorString(e));
  return ADAPTRA_OK;
}

}  // namespace adaptra
