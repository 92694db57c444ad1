// HBM-bound kernels of the stage path: LayerNorm fwd / bwd-input / param
// grads, causal softmax, attention row-dot D = rowsum(dO * O), column sums
// (bias grads), MSE loss + dy seed, and the 16B-vector copy used by the P2P
// link and the stash.  Warp-per-row with 16-byte vector accesses where the row
// is aligned; fp32 arithmetic everywhere.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "../../../include/adaptra.h"
#include "../prof.h"
#include "../util.h"
#include "common.cuh"
#include "kernels.h"

namespace adaptra {

constexpr float kLnEps = 1e-5f;

template <typename T>
__device__ __forceinline__ void load8(const T* p, float* v);
template <>
__device__ __forceinline__ void load8<float>(const float* p, float* v) {
  float4 a = *reinterpret_cast<const float4*>(p);
  float4 b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
template <>
__device__ __forceinline__ void load8<bf16>(const bf16* p, float* v) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  float2 f;
  f = unpack_bf16x2(u.x); v[0] = f.x; v[1] = f.y;
  f = unpack_bf16x2(u.y); v[2] = f.x; v[3] = f.y;
  f = unpack_bf16x2(u.z); v[4] = f.x; v[5] = f.y;
  f = unpack_bf16x2(u.w); v[6] = f.x; v[7] = f.y;
}
template <typename T>
__device__ __forceinline__ void store8(T* p, const float* v);
template <>
__device__ __forceinline__ void store8<float>(float* p, const float* v) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}
template <>
__device__ __forceinline__ void store8<bf16>(bf16* p, const float* v) {
  uint4 u;
  u.x = pack_bf16x2(v[0], v[1]);
  u.y = pack_bf16x2(v[2], v[3]);
  u.z = pack_bf16x2(v[4], v[5]);
  u.w = pack_bf16x2(v[6], v[7]);
  *reinterpret_cast<uint4*>(p) = u;
}

// ---------------------------------------------------------------- LayerNorm
// h = gamma * (x - mean) * rstd + beta; one warp per row, d % 8 == 0.
template <typename T>
__global__ void ln_fwd_kernel(const T* __restrict__ x, const float* __restrict__ g, const float* __restrict__ b,
                              T* __restrict__ h, float* __restrict__ mean_out, float* __restrict__ rstd_out, int R,
                              int d) {
  int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x % 32;
  if (row >= R) return;
  const T* xr = x + (long)row * d;
  float s = 0.f;
  for (int c = lane * 8; c < d; c += 256) {
    float v[8];
    load8(xr + c, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[j];
  }
  const float mu = warp_sum(s) / d;
  float q = 0.f;
  for (int c = lane * 8; c < d; c += 256) {
    float v[8];
    load8(xr + c, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) q += (v[j] - mu) * (v[j] - mu);
  }
  const float rs = rsqrtf(warp_sum(q) / d + kLnEps);
  T* hr = h + (long)row * d;
  for (int c = lane * 8; c < d; c += 256) {
    float v[8], o[8];
    load8(xr + c, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = (v[j] - mu) * rs * g[c + j] + b[c + j];
    store8(hr + c, o);
  }
  if (lane == 0) {
    mean_out[row] = mu;
    rstd_out[row] = rs;
  }
}

// dx = dres + rstd * (gd - mean(gd) - xhat * mean(gd * xhat)), gd = dh * gamma.
template <typename T>
__global__ void ln_bwd_kernel(const T* __restrict__ dh, const T* __restrict__ x, const float* __restrict__ mean,
                              const float* __restrict__ rstd, const float* __restrict__ g, const T* __restrict__ dres,
                              T* __restrict__ dx, int R, int d) {
  int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x % 32;
  if (row >= R) return;
  const T* dr = dh + (long)row * d;
  const T* xr = x + (long)row * d;
  const float mu = mean[row], rs = rstd[row];
  float s1 = 0.f, s2 = 0.f;
  for (int c = lane * 8; c < d; c += 256) {
    float a[8], v[8];
    load8(dr + c, a);
    load8(xr + c, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float gd = a[j] * g[c + j];
      float xh = (v[j] - mu) * rs;
      s1 += gd;
      s2 += gd * xh;
    }
  }
  s1 = warp_sum(s1) / d;
  s2 = warp_sum(s2) / d;
  for (int c = lane * 8; c < d; c += 256) {
    float a[8], v[8], r[8], o[8];
    load8(dr + c, a);
    load8(xr + c, v);
    load8(dres + (long)row * d + c, r);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float gd = a[j] * g[c + j];
      float xh = (v[j] - mu) * rs;
      o[j] = r[j] + rs * (gd - s1 - xh * s2);
    }
    store8(dx + (long)row * d + c, o);
  }
}

// Column reductions: out[c] += sum_r f(r, c).  Block = 32 x 8 threads over a
// 32-column strip and a chunk of rows; fp32 partials, one atomicAdd per column
// per block.
template <typename T, bool LN>
__global__ void colsum_kernel(const T* __restrict__ y, const T* __restrict__ x, const float* __restrict__ mean,
                              const float* __restrict__ rstd, float* __restrict__ out_a, float* __restrict__ out_b,
                              int R, int N, int rows_per_block) {
  __shared__ float sa[8][33], sb[8][33];
  int c = blockIdx.x * 32 + threadIdx.x;
  int r0 = blockIdx.y * rows_per_block;
  int r1 = min(R, r0 + rows_per_block);
  float a = 0.f, b = 0.f;
  if (c < N) {
    for (int r = r0 + threadIdx.y; r < r1; r += 8) {
      float v = to_f(y[(long)r * N + c]);
      if (LN) {
        float xh = (to_f(x[(long)r * N + c]) - mean[r]) * rstd[r];
        a += v * xh;
        b += v;
      } else {
        a += v;
      }
    }
  }
  sa[threadIdx.y][threadIdx.x] = a;
  sb[threadIdx.y][threadIdx.x] = b;
  __syncthreads();
  if (threadIdx.y == 0 && c < N) {
    float ta = 0.f, tb = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      ta += sa[k][threadIdx.x];
      tb += sb[k][threadIdx.x];
    }
    atomicAdd(out_a + c, ta);
    if (LN) atomicAdd(out_b + c, tb);
  }
}

// Register-resident variants (one warp per row, the row kept in registers:
// V 8-element vectors per lane, d = 256 V): one HBM read of each input.
template <typename T, int V>
__global__ void __launch_bounds__(128) ln_fwd_reg_kernel(const T* __restrict__ x, const float* __restrict__ g,
                                                         const float* __restrict__ b, T* __restrict__ h,
                                                         float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                                         int R, int d) {
  int row = blockIdx.x * 4 + threadIdx.x / 32;
  int lane = threadIdx.x % 32;
  if (row >= R) return;
  const T* xr = x + (long)row * d;
  float v[V][8];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    load8(xr + k * 256 + lane * 8, v[k]);
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[k][j];
  }
  const float mu = warp_sum(s) / d;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < V; ++k)
#pragma unroll
    for (int j = 0; j < 8; ++j) q += (v[k][j] - mu) * (v[k][j] - mu);
  const float rs = rsqrtf(warp_sum(q) / d + kLnEps);
  T* hr = h + (long)row * d;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int c = k * 256 + lane * 8;
    float gg[8], bb[8], o[8];
    *reinterpret_cast<float4*>(gg) = *reinterpret_cast<const float4*>(g + c);
    *reinterpret_cast<float4*>(gg + 4) = *reinterpret_cast<const float4*>(g + c + 4);
    *reinterpret_cast<float4*>(bb) = *reinterpret_cast<const float4*>(b + c);
    *reinterpret_cast<float4*>(bb + 4) = *reinterpret_cast<const float4*>(b + c + 4);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = (v[k][j] - mu) * rs * gg[j] + bb[j];
    store8(hr + c, o);
  }
  if (lane == 0) {
    mean_out[row] = mu;
    rstd_out[row] = rs;
  }
}

template <typename T, int V>
__global__ void __launch_bounds__(128) ln_bwd_reg_kernel(const T* __restrict__ dh, const T* __restrict__ x,
                                                         const float* __restrict__ mean, const float* __restrict__ rstd,
                                                         const float* __restrict__ g, const T* __restrict__ dres,
                                                         T* __restrict__ dx, int R, int d) {
  int row = blockIdx.x * 4 + threadIdx.x / 32;
  int lane = threadIdx.x % 32;
  if (row >= R) return;
  const float mu = mean[row], rs = rstd[row];
  float gd[V][8], xh[V][8];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int c = k * 256 + lane * 8;
    float a[8], gg[8];
    load8(dh + (long)row * d + c, a);
    load8(x + (long)row * d + c, xh[k]);
    *reinterpret_cast<float4*>(gg) = *reinterpret_cast<const float4*>(g + c);
    *reinterpret_cast<float4*>(gg + 4) = *reinterpret_cast<const float4*>(g + c + 4);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      gd[k][j] = a[j] * gg[j];
      xh[k][j] = (xh[k][j] - mu) * rs;
      s1 += gd[k][j];
      s2 += gd[k][j] * xh[k][j];
    }
  }
  s1 = warp_sum(s1) / d;
  s2 = warp_sum(s2) / d;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int c = k * 256 + lane * 8;
    float r[8], o[8];
    load8(dres + (long)row * d + c, r);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = r[j] + rs * (gd[k][j] - s1 - xh[k][j] * s2);
    store8(dx + (long)row * d + c, o);
  }
}

// Column sums with 16 B loads: block = 256 threads over 64 columns x 256 rows
// (8 column groups of 8 x 32 row lanes), shared-memory reduction, one
// atomicAdd per column per block.  LN: out_a += dh * xhat, out_b += dh.
template <typename T, bool LN>
__global__ void __launch_bounds__(256) colsum_vec_kernel(const T* __restrict__ y, const T* __restrict__ x,
                                                         const float* __restrict__ mean,
                                                         const float* __restrict__ rstd, float* __restrict__ out_a,
                                                         float* __restrict__ out_b, int R, int N) {
  __shared__ float sa[32][65], sb[32][65];
  const int cg = threadIdx.x & 7, rl = threadIdx.x >> 3;
  const int c0 = blockIdx.x * 64 + cg * 8;
  const int r0 = blockIdx.y * 256;
  float a[8] = {}, bsum[8] = {};
  if (c0 < N) {
    for (int r = r0 + rl; r < min(R, r0 + 256); r += 32) {
      float v[8];
      load8(y + (long)r * N + c0, v);
      if (LN) {
        float xv[8];
        load8(x + (long)r * N + c0, xv);
        const float mu = mean[r], rs = rstd[r];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          a[j] += v[j] * (xv[j] - mu) * rs;
          bsum[j] += v[j];
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] += v[j];
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    sa[rl][cg * 8 + j] = a[j];
    if (LN) sb[rl][cg * 8 + j] = bsum[j];
  }
  __syncthreads();
  if (threadIdx.x < 64) {
    const int c = blockIdx.x * 64 + threadIdx.x;
    float ta = 0.f, tb = 0.f;
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      ta += sa[k][threadIdx.x];
      if (LN) tb += sb[k][threadIdx.x];
    }
    if (c < N) {
      atomicAdd(out_a + c, ta);
      if (LN) atomicAdd(out_b + c, tb);
    }
  }
}

// Deterministic column sums (bias and LN parameter gradients of W), 16 B
// loads: block = 256 threads over 64 columns x 256 rows (8 column groups of
// 8 x 32 row lanes, the 8 rows of a thread loaded before any is summed); the
// block's 64 sums go to part[by][c]; the last block of a column strip (ticket
// on cnt[bx], reset by it) adds the strip's partials in row-block order to
// out (out += ...; one writer per column), so the result is bit-reproducible
// and independent of block scheduling.  LN: out_a += dh * xhat, out_b += dh.
template <typename T, bool LN>
__device__ __forceinline__ void colsum_block(const T* __restrict__ y, const T* __restrict__ x,
                                             const float* __restrict__ mean, const float* __restrict__ rstd,
                                             float* __restrict__ out_a, float* __restrict__ out_b, int R, int N, int bx,
                                             int by, int nby, float* __restrict__ part, unsigned* __restrict__ cnt,
                                             float (*sa)[65], float (*sb)[65], bool* last) {
  const int cg = threadIdx.x & 7, rl = threadIdx.x >> 3;
  const int c0 = bx * 64 + cg * 8;
  const int r0 = by * 256;
  float a[8] = {}, bsum[8] = {};
  if (c0 < N) {
    float v[8][8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = r0 + rl + 32 * k;
      if (r < R) {
        load8(y + (long)r * N + c0, v[k]);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[k][j] = 0.f;
      }
    }
    if (LN) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int r = r0 + rl + 32 * k;
        if (r >= R) continue;
        float xv[8];
        load8(x + (long)r * N + c0, xv);
        const float mu = mean[r], rs = rstd[r];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          a[j] += v[k][j] * (xv[j] - mu) * rs;
          bsum[j] += v[k][j];
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] += v[k][j];
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    sa[rl][cg * 8 + j] = a[j];
    if (LN) sb[rl][cg * 8 + j] = bsum[j];
  }
  __syncthreads();
  const int c = bx * 64 + threadIdx.x;
  if (threadIdx.x < 64) {
    float ta = 0.f, tb = 0.f;
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      ta += sa[k][threadIdx.x];
      if (LN) tb += sb[k][threadIdx.x];
    }
    if (c < N) {
      part[(size_t)by * N + c] = ta;
      if (LN) part[(size_t)(nby + by) * N + c] = tb;
    }
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) *last = atomicAdd(&cnt[bx], 1u) == (unsigned)nby - 1;
  __syncthreads();
  if (!*last) return;
  __threadfence();
  if (threadIdx.x < 64 && c < N) {
    float ta = 0.f, tb = 0.f;
    for (int k = 0; k < nby; ++k) {
      ta += __ldcg(part + (size_t)k * N + c);
      if (LN) tb += __ldcg(part + (size_t)(nby + k) * N + c);
    }
    out_a[c] += ta;
    if (LN) out_b[c] += tb;
  }
  if (threadIdx.x == 0) cnt[bx] = 0u;
}

template <typename T, bool LN>
__global__ void __launch_bounds__(256) colsum_det_kernel(const T* __restrict__ y, const T* __restrict__ x,
                                                         const float* __restrict__ mean,
                                                         const float* __restrict__ rstd, float* __restrict__ out_a,
                                                         float* __restrict__ out_b, int R, int N,
                                                         float* __restrict__ part, unsigned* __restrict__ cnt) {
  __shared__ float sa[32][65], sb[32][65];
  __shared__ bool last;
  colsum_block<T, LN>(y, x, mean, rstd, out_a, out_b, R, N, blockIdx.x, blockIdx.y, gridDim.y, part, cnt, sa, sb,
                      &last);
}

// ---------------------------------------------------------------- attention
// Row i of batch z: P[i, j] = exp(S[i, j] - max) / sum over j <= i; zeros for
// i < j < roundup(i + 1, 128) so that tile-granular consumers read zeros.
template <typename T>
__global__ void softmax_causal_kernel(const float* __restrict__ S, T* __restrict__ P, int Z, int Tn) {
  long rowg = (long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x % 32;
  if (rowg >= (long)Z * Tn) return;
  int i = (int)(rowg % Tn);
  const float* s = S + rowg * Tn;
  T* p = P + rowg * Tn;
  float m = -INFINITY;
  for (int j = lane; j <= i; j += 32) m = fmaxf(m, s[j]);
  m = warp_max(m);
  float sum = 0.f;
  for (int j = lane; j <= i; j += 32) sum += __expf(s[j] - m);
  sum = warp_sum(sum);
  const float inv = 1.f / sum;
  int jend = min(Tn, ((i + 1 + 127) / 128) * 128);
  for (int j = lane; j < jend; j += 32) p[j] = from_f<T>(j <= i ? __expf(s[j] - m) * inv : 0.f);
}

// D[z, i] = sum_c dO[i, c] * O[i, c] over the head's dh columns (softmax bwd).
template <typename T>
__global__ void attn_rowdot_kernel(const T* __restrict__ dO, const T* __restrict__ O, float* __restrict__ D, int b,
                                   int H, int Tn, int dh, int ld) {
  long w = (long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x % 32;
  if (w >= (long)b * H * Tn) return;
  int i = (int)(w % Tn);
  long zh = w / Tn;
  int h = (int)(zh % H);
  int s = (int)(zh / H);
  long off = ((long)s * Tn + i) * ld + (long)h * dh;
  float acc = 0.f;
  for (int c = lane * 8; c < dh; c += 256) {
    float a[8], v[8];
    load8(dO + off + c, a);
    load8(O + off + c, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += a[j] * v[j];
  }
  acc = warp_sum(acc);
  if (lane == 0) D[w] = acc;
}

// ---------------------------------------------------------------- loss (R19)
// L_j = (1/(R d)) sum 1/2 (y - tgt)^2, loss_acc += L_j / N;  dy = (y - tgt)/(N R d).
template <typename T>
__global__ void mse_kernel(const T* __restrict__ y, const float* __restrict__ tgt, T* __restrict__ dy,
                           float* __restrict__ part, long n, float inv_n_total, float inv_loss) {
  __shared__ float red[32];
  float acc = 0.f;
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
    float e = to_f(y[k]) - tgt[k];
    acc += 0.5f * e * e;
    dy[k] = from_f<T>(e * inv_n_total);
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = v * inv_loss;
  }
}
// fixed-order sum of the per-block partials (one block of 256 threads)
__global__ void mse_sum_kernel(const float* __restrict__ part, int n, float* __restrict__ loss_acc) {
  __shared__ float red[8];
  float acc = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += part[i];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float v = 0.f;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) v += red[w];
    *loss_acc += v;
  }
}

// ---------------------------------------------------------------- copy
__global__ void copy16_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, long n16) {
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < n16; k += (long)gridDim.x * blockDim.x)
    dst[k] = src[k];
}

// ================================================================ launchers
static int launch_check(const char* what) {
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ADAPTRA_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return ADAPTRA_OK;
}

template <typename T>
int ln_fwd(const T* x, const float* g, const float* b, T* h, float* mean, float* rstd, int R, int d, cudaStream_t st) {
  const dim3 gr((R + 3) / 4);
  switch (d % 256 ? 0 : d / 256) {
    case 1: ln_fwd_reg_kernel<T, 1><<<gr, 128, 0, st>>>(x, g, b, h, mean, rstd, R, d); break;
    case 2: ln_fwd_reg_kernel<T, 2><<<gr, 128, 0, st>>>(x, g, b, h, mean, rstd, R, d); break;
    case 4: ln_fwd_reg_kernel<T, 4><<<gr, 128, 0, st>>>(x, g, b, h, mean, rstd, R, d); break;
    case 8: ln_fwd_reg_kernel<T, 8><<<gr, 128, 0, st>>>(x, g, b, h, mean, rstd, R, d); break;
    case 16: ln_fwd_reg_kernel<T, 16><<<gr, 128, 0, st>>>(x, g, b, h, mean, rstd, R, d); break;
    default: ln_fwd_kernel<T><<<(R + 7) / 8, 256, 0, st>>>(x, g, b, h, mean, rstd, R, d);
  }
  return launch_check("ln_fwd");
}
template <typename T>
int ln_bwd(const T* dh, const T* x, const float* mean, const float* rstd, const float* g, const T* dres, T* dx, int R,
           int d, cudaStream_t st) {
  const dim3 gr((R + 3) / 4);
  switch (d % 256 ? 0 : d / 256) {
    case 1: ln_bwd_reg_kernel<T, 1><<<gr, 128, 0, st>>>(dh, x, mean, rstd, g, dres, dx, R, d); break;
    case 2: ln_bwd_reg_kernel<T, 2><<<gr, 128, 0, st>>>(dh, x, mean, rstd, g, dres, dx, R, d); break;
    case 4: ln_bwd_reg_kernel<T, 4><<<gr, 128, 0, st>>>(dh, x, mean, rstd, g, dres, dx, R, d); break;
    case 8: ln_bwd_reg_kernel<T, 8><<<gr, 128, 0, st>>>(dh, x, mean, rstd, g, dres, dx, R, d); break;
    case 16: ln_bwd_reg_kernel<T, 16><<<gr, 128, 0, st>>>(dh, x, mean, rstd, g, dres, dx, R, d); break;
    default: ln_bwd_kernel<T><<<(R + 7) / 8, 256, 0, st>>>(dh, x, mean, rstd, g, dres, dx, R, d);
  }
  return launch_check("ln_bwd");
}
template <typename T>
int ln_param_grad(const T* dh, const T* x, const float* mean, const float* rstd, float* dg, float* db, int R, int d,
                  cudaStream_t st, float* part, unsigned* cnt) {
  if (d % 8 == 0 && part) {
    colsum_det_kernel<T, true>
        <<<dim3((d + 63) / 64, (R + 255) / 256), 256, 0, st>>>(dh, x, mean, rstd, dg, db, R, d, part, cnt);
  } else if (d % 8 == 0) {
    colsum_vec_kernel<T, true><<<dim3((d + 63) / 64, (R + 255) / 256), 256, 0, st>>>(dh, x, mean, rstd, dg, db, R, d);
  } else {
    int rpb = 256;
    dim3 grid((d + 31) / 32, (R + rpb - 1) / rpb);
    colsum_kernel<T, true><<<grid, dim3(32, 8), 0, st>>>(dh, x, mean, rstd, dg, db, R, d, rpb);
  }
  return launch_check("ln_param_grad");
}
template <typename T>
int col_sum(const T* y, float* out, int R, int N, cudaStream_t st, float* part, unsigned* cnt) {
  if (N % 8 == 0 && part) {
    colsum_det_kernel<T, false><<<dim3((N + 63) / 64, (R + 255) / 256), 256, 0, st>>>(
        y, nullptr, nullptr, nullptr, out, nullptr, R, N, part, cnt);
  } else if (N % 8 == 0) {
    colsum_vec_kernel<T, false>
        <<<dim3((N + 63) / 64, (R + 255) / 256), 256, 0, st>>>(y, nullptr, nullptr, nullptr, out, nullptr, R, N);
  } else {
    int rpb = 256;
    dim3 grid((N + 31) / 32, (R + rpb - 1) / rpb);
    colsum_kernel<T, false><<<grid, dim3(32, 8), 0, st>>>(y, nullptr, nullptr, nullptr, out, nullptr, R, N, rpb);
  }
  return launch_check("col_sum");
}
template <typename T>
int softmax_causal(const float* S, T* P, int Z, int Tn, cudaStream_t st) {
  long rows = (long)Z * Tn;
  softmax_causal_kernel<T><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(S, P, Z, Tn);
  return launch_check("softmax_causal");
}
template <typename T>
int attn_rowdot(const T* dO, const T* O, float* D, int b, int H, int Tn, int dh, int ld, cudaStream_t st) {
  long w = (long)b * H * Tn;
  attn_rowdot_kernel<T><<<(unsigned)((w + 7) / 8), 256, 0, st>>>(dO, O, D, b, H, Tn, dh, ld);
  return launch_check("attn_rowdot");
}
template <typename T>
int mse_loss(const T* y, const float* tgt, T* dy, float* loss_acc, float* part, long n, int n_mb, cudaStream_t st) {
  float inv_total = 1.f / ((float)n_mb * (float)n);
  float inv_loss = 1.f / ((float)n * (float)n_mb);
  int blocks = (int)std::min<long>(kMseMaxBlocks, (n + 255) / 256);
  mse_kernel<T><<<blocks, 256, 0, st>>>(y, tgt, dy, part, n, inv_total, inv_loss);
  mse_sum_kernel<<<1, 256, 0, st>>>(part, blocks, loss_acc);
  return launch_check("mse_loss");
}
int copy_async(void* dst, const void* src, long bytes, cudaStream_t st) {
  if (bytes % 16 || ((uintptr_t)dst | (uintptr_t)src) % 16) {
    ADAPTRA_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
    return ADAPTRA_OK;
  }
  long n16 = bytes / 16;
  int blocks = (int)std::min<long>(32, (n16 + 511) / 512);
  copy16_kernel<<<blocks, 512, 0, st>>>((const uint4*)src, (uint4*)dst, n16);
  return launch_check("copy16");
}

// All column sums of a W op (bias gradients db += sum_rows dY and LN
// parameter gradients) in one launch: job j owns blocks [start_j, start_j +
// nbx_j * nby); each block is colsum_vec_kernel's 64 columns x 256 rows.
template <typename T>
__global__ void __launch_bounds__(256) colsum_grouped_kernel(const ColsumGroup g) {
  int j = 0;
  while (j + 1 < g.n && (int)blockIdx.x >= g.job[j + 1].start) ++j;
  const ColsumJob& J = g.job[j];
  const int nby = (g.R + 255) / 256;
  const int b = blockIdx.x - J.start, bx = b % J.nbx, by = b / J.nbx;
  __shared__ float sa[32][65], sb[32][65];
  __shared__ bool last;
  if (J.part) {
    if (J.ln)
      colsum_block<T, true>((const T*)J.y, (const T*)J.x, J.mean, J.rstd, J.out_a, J.out_b, g.R, J.N, bx, by, nby,
                            J.part, J.cnt, sa, sb, &last);
    else
      colsum_block<T, false>((const T*)J.y, nullptr, nullptr, nullptr, J.out_a, nullptr, g.R, J.N, bx, by, nby,
                             J.part, J.cnt, sa, sb, &last);
    return;
  }
  // atomic fallback (no workspace): one atomicAdd per column per block
  const T* __restrict__ y = (const T*)J.y;
  const T* __restrict__ x = (const T*)J.x;
  const int N = J.N, R = g.R;
  const int cg = threadIdx.x & 7, rl = threadIdx.x >> 3;
  const int c0 = bx * 64 + cg * 8;
  const int r0 = by * 256;
  float a[8] = {}, bsum[8] = {};
  if (c0 < N) {
    for (int r = r0 + rl; r < min(R, r0 + 256); r += 32) {
      float v[8];
      load8(y + (long)r * N + c0, v);
      if (J.ln) {
        float xv[8];
        load8(x + (long)r * N + c0, xv);
        const float mu = J.mean[r], rs = J.rstd[r];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          a[k] += v[k] * (xv[k] - mu) * rs;
          bsum[k] += v[k];
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] += v[k];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    sa[rl][cg * 8 + k] = a[k];
    sb[rl][cg * 8 + k] = bsum[k];
  }
  __syncthreads();
  if (threadIdx.x < 64) {
    const int c = bx * 64 + threadIdx.x;
    float ta = 0.f, tb = 0.f;
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      ta += sa[k][threadIdx.x];
      tb += sb[k][threadIdx.x];
    }
    if (c < N) {
      atomicAdd(J.out_a + c, ta);
      if (J.ln) atomicAdd(J.out_b + c, tb);
    }
  }
}
template <typename T>
int colsum_grouped(const ColsumJob* jobs, int n, int R, cudaStream_t st, float* part, unsigned* cnt, long part_cap,
                   long cnt_cap) {
  const int nby = (R + 255) / 256;
  for (int i0 = 0; i0 < n; i0 += kMaxColsum) {
    ColsumGroup g{};
    g.n = std::min(kMaxColsum, n - i0);
    g.R = R;
    int blocks = 0;
    long poff = 0, coff = 0;  // each job its own partials and tickets (the group's jobs run concurrently)
    for (int k = 0; k < g.n; ++k) {
      g.job[k] = jobs[i0 + k];
      if (g.job[k].N % 8) return set_error(ADAPTRA_EINVAL, "colsum_grouped: N % 8 != 0");
      g.job[k].nbx = (g.job[k].N + 63) / 64;
      g.job[k].start = blocks;
      blocks += g.job[k].nbx * nby;
      g.job[k].part = nullptr;
      g.job[k].cnt = nullptr;
      if (part) {
        const long need = 2L * nby * g.job[k].N;
        if (poff + need > part_cap || coff + g.job[k].nbx > cnt_cap)
          return set_error(ADAPTRA_ENOMEM, "colsum_grouped: workspace too small");
        g.job[k].part = part + poff;
        g.job[k].cnt = cnt + coff;
        poff += need;
        coff += g.job[k].nbx;
      }
    }
    if (blocks == 0) continue;
    colsum_grouped_kernel<T><<<blocks, 256, 0, st>>>(g);
    int rc = launch_check("colsum_grouped");
    if (rc) return rc;
  }
  return ADAPTRA_OK;
}

#define INST(T)                                                                                                   \
  template int ln_fwd<T>(const T*, const float*, const float*, T*, float*, float*, int, int, cudaStream_t);       \
  template int ln_bwd<T>(const T*, const T*, const float*, const float*, const float*, const T*, T*, int, int,    \
                         cudaStream_t);                                                                           \
  template int ln_param_grad<T>(const T*, const T*, const float*, const float*, float*, float*, int, int,        \
                                cudaStream_t, float*, unsigned*);                                                 \
  template int col_sum<T>(const T*, float*, int, int, cudaStream_t, float*, unsigned*);                           \
  template int softmax_causal<T>(const float*, T*, int, int, cudaStream_t);                                       \
  template int attn_rowdot<T>(const T*, const T*, float*, int, int, int, int, int, cudaStream_t);                 \
  template int colsum_grouped<T>(const ColsumJob*, int, int, cudaStream_t, float*, unsigned*, long, long);        \
  template int mse_loss<T>(const T*, const float*, T*, float*, float*, long, int, cudaStream_t);
INST(float)
INST(bf16)

}  // namespace adaptra
