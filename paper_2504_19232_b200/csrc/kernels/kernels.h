// Launch wrappers of the stage kernels (csrc/kernels/*.cu).  Host-callable.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../../include/adaptra.h"

namespace adaptra {
typedef __nv_bfloat16 bf16;

int gemm_tc(const adaptra_gemm_desc_t& g, cudaStream_t st);
// Independent products in one persistent launch (W op's dW += X^T dY);
// falls back to one gemm_tc per product outside its specialisation.
// more[0..n_more) (optional, n entries each, n_more <= 3): further K segments --
// product i becomes C_i += A_i^T B_i + sum_m A_{m,i}^T B_{m,i} in one K loop
// (same M, N, K, C; the W of up to four slots).  dbias[i] (optional, fp32,
// M_i entries): db_i += the column sums of A_i over all K segments, summed
// from the staged dY tiles inside the same launch; *fused says whether that
// happened (false on the per-product fallback: the caller sums instead).
int gemm_tc_grouped(const adaptra_gemm_desc_t* gs, int n, cudaStream_t st,
                    const adaptra_gemm_desc_t* const* more = nullptr, int n_more = 0, float* const* dbias = nullptr,
                    bool* fused = nullptr);
int gemm_simt(const adaptra_gemm_desc_t& g, cudaStream_t st);

template <typename T>
int ln_fwd(const T* x, const float* g, const float* b, T* h, float* mean, float* rstd, int R, int d, cudaStream_t st);
template <typename T>
int ln_bwd(const T* dh, const T* x, const float* mean, const float* rstd, const float* g, const T* dres, T* dx, int R,
           int d, cudaStream_t st);
template <typename T>
// part / cnt (optional): deterministic two-level reduction workspace, part
// [2 * ceil(R / 256) * N] fp32, cnt [ceil(N / 64)] zeroed once (self-resetting);
// without them one atomicAdd per column per block (order not reproducible)
int ln_param_grad(const T* dh, const T* x, const float* mean, const float* rstd, float* dg, float* db, int R, int d,
                  cudaStream_t st, float* part = nullptr, unsigned* cnt = nullptr);
template <typename T>
int col_sum(const T* y, float* out, int R, int N, cudaStream_t st, float* part = nullptr, unsigned* cnt = nullptr);
// One launch for many column sums (a W op's bias and LN parameter gradients):
// ln = 0: out_a[c] += sum_r y[r,c];  ln = 1: out_a[c] += sum_r y (x - mean) rstd,
// out_b[c] += sum_r y.  y, x row-major [R, N], N % 8 == 0.
struct ColsumJob {
  const void* y;
  const void* x;
  const float* mean;
  const float* rstd;
  float* out_a;
  float* out_b;
  int N, ln;
  int start, nbx;  // filled by colsum_grouped
  float* part;     // filled by colsum_grouped: [2][nby][N] partials in the workspace
  unsigned* cnt;   // [nbx] tickets (zero, self-resetting)
};
constexpr int kMaxColsum = 48;
struct ColsumGroup {
  int n, R;
  ColsumJob job[kMaxColsum];
};
template <typename T>
// part / cnt: deterministic workspace (colsum_grouped_ws_floats / _tickets);
// NULL = one atomicAdd per column per block
int colsum_grouped(const ColsumJob* jobs, int n, int R, cudaStream_t st, float* part = nullptr, unsigned* cnt = nullptr,
                   long part_cap = 0, long cnt_cap = 0);
template <typename T>
int softmax_causal(const float* S, T* P, int Z, int Tn, cudaStream_t st);
template <typename T>
int attn_rowdot(const T* dO, const T* O, float* D, int b, int H, int Tn, int dh, int ld, cudaStream_t st);
// MSE loss + dy seed; per-block partial sums go to part[kMseMaxBlocks] and a
// one-block kernel adds them to *loss_acc in a fixed order (reproducible loss).
constexpr int kMseMaxBlocks = 1184;
template <typename T>
int mse_loss(const T* y, const float* tgt, T* dy, float* loss_acc, float* part, long n, int n_mb, cudaStream_t st);
int copy_async(void* dst, const void* src, long bytes, cudaStream_t st);
// fused causal attention (bf16, head dim 128): attn_tc.cu
int attn_fwd_tc(const bf16* qkv, bf16* o, float* lse, int b, int H, int T, int d, cudaStream_t st);
int attn_bwd_tc(const bf16* qkv, const bf16* dO, const float* lse, const float* D, bf16* dqkv, float* dq_acc, int b,
                int H, int T, int d, cudaStream_t st);
}  // namespace adaptra
