// Fused GEMM epilogues shared by the tcgen05 kernel and the SIMT parity kernel.
// One thread handles one output row m and a run of consecutive columns.
#pragma once
#include "../../../include/adaptra.h"
#include "common.cuh"

namespace adaptra {

struct EpiCtx {
  int epi;
  float alpha;
  int M, N;
  char* C;
  long ldc;
  char* aux;
  long ldaux;
  const char* R;
  long ldr;
  const float* bias;
  const float* rowv;
};

// Batch-resolved epilogue context for batch z.
template <typename T>
__device__ __forceinline__ EpiCtx make_epi(const adaptra_gemm_desc_t& g, int z) {
  EpiCtx e;
  int z1 = z / g.zdiv, z2 = z % g.zdiv;
  e.epi = g.epi;
  e.alpha = g.alpha;
  e.M = g.M;
  e.N = g.N;
  bool f32out = (g.epi == ADAPTRA_EPI_ACC_F32 || g.epi == ADAPTRA_EPI_STORE_F32);
  long csz = f32out ? 4 : (long)sizeof(T);
  e.C = (char*)g.C + (z1 * g.c_1 + z2 * g.c_2) * csz;
  e.ldc = g.ldc;
  e.aux = g.aux ? (char*)g.aux + (z1 * g.aux_1 + z2 * g.aux_2) * (long)sizeof(T) : nullptr;
  e.ldaux = g.ldaux;
  e.R = (const char*)g.R;
  e.ldr = g.ldr;
  e.bias = g.bias;
  e.rowv = g.rowv ? g.rowv + (z1 * g.rowv_1 + z2 * g.rowv_2) : nullptr;
  return e;
}

// Apply the epilogue to v[0..n) = accumulator values of row m, columns n0..n0+n.
template <typename T, int NV>
__device__ __forceinline__ void epi_row(const EpiCtx& e, int m, int n0, float (&v)[NV]) {
  if (m >= e.M) return;
  const int nlim = e.N - n0;
  switch (e.epi) {
    case ADAPTRA_EPI_STORE: {
      T* c = (T*)e.C + (long)m * e.ldc + n0;
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (j < nlim) c[j] = from_f<T>(e.alpha * v[j] + (e.bias ? e.bias[n0 + j] : 0.f));
    } break;
    case ADAPTRA_EPI_GELU: {
      T* c = (T*)e.C + (long)m * e.ldc + n0;
      T* a = (T*)e.aux + (long)m * e.ldaux + n0;
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (j < nlim) {
          float x = v[j] + (e.bias ? e.bias[n0 + j] : 0.f);
          T xs = from_f<T>(x);
          a[j] = xs;
          c[j] = from_f<T>(gelu_f(to_f(xs)));
        }
    } break;
    case ADAPTRA_EPI_RESID: {
      T* c = (T*)e.C + (long)m * e.ldc + n0;
      const T* r = (const T*)e.R + (long)m * e.ldr + n0;
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (j < nlim) c[j] = from_f<T>(v[j] + (e.bias ? e.bias[n0 + j] : 0.f) + to_f(r[j]));
    } break;
    case ADAPTRA_EPI_DGELU: {
      T* c = (T*)e.C + (long)m * e.ldc + n0;
      const T* a = (const T*)e.aux + (long)m * e.ldaux + n0;
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (j < nlim) c[j] = from_f<T>(v[j] * gelu_grad_f(to_f(a[j])));
    } break;
    case ADAPTRA_EPI_ACC_F32: {
      float* c = (float*)e.C + (long)m * e.ldc + n0;
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (j < nlim) c[j] += e.alpha * v[j];
    } break;
    case ADAPTRA_EPI_STORE_F32: {
      float* c = (float*)e.C + (long)m * e.ldc + n0;
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (j < nlim) c[j] = e.alpha * v[j];
    } break;
    case ADAPTRA_EPI_DSOFTMAX: {
      T* c = (T*)e.C + (long)m * e.ldc + n0;
      const T* p = (const T*)e.aux + (long)m * e.ldaux + n0;
      float D = e.rowv[m];
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (j < nlim) c[j] = from_f<T>(to_f(p[j]) * (v[j] - D) * e.alpha);
    } break;
  }
}

// Vectorised bf16 variant for a full run of NV (multiple of 8) in-range, 16B-aligned columns.
__device__ __forceinline__ void st_bf16x8(bf16* p, const float* v) {
  uint4 u;
  u.x = pack_bf16x2(v[0], v[1]);
  u.y = pack_bf16x2(v[2], v[3]);
  u.z = pack_bf16x2(v[4], v[5]);
  u.w = pack_bf16x2(v[6], v[7]);
  *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ void ld_bf16x8(const bf16* p, float* v) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  float2 f;
  f = unpack_bf16x2(u.x); v[0] = f.x; v[1] = f.y;
  f = unpack_bf16x2(u.y); v[2] = f.x; v[3] = f.y;
  f = unpack_bf16x2(u.z); v[4] = f.x; v[5] = f.y;
  f = unpack_bf16x2(u.w); v[6] = f.x; v[7] = f.y;
}

template <int NV>
__device__ __forceinline__ void epi_rowN_bf16_fast(const EpiCtx& e, int m, int n0, float (&v)[NV]) {
  switch (e.epi) {
    case ADAPTRA_EPI_STORE: {
      bf16* c = (bf16*)e.C + (long)m * e.ldc + n0;
      if (e.bias) {
#pragma unroll
        for (int j = 0; j < NV; j += 4) {
          float4 b = *reinterpret_cast<const float4*>(e.bias + n0 + j);
          v[j] = e.alpha * v[j] + b.x; v[j + 1] = e.alpha * v[j + 1] + b.y;
          v[j + 2] = e.alpha * v[j + 2] + b.z; v[j + 3] = e.alpha * v[j + 3] + b.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < NV; ++j) v[j] *= e.alpha;
      }
#pragma unroll
      for (int j = 0; j < NV; j += 8) st_bf16x8(c + j, v + j);
    } break;
    case ADAPTRA_EPI_GELU: {
      bf16* c = (bf16*)e.C + (long)m * e.ldc + n0;
      bf16* a = (bf16*)e.aux + (long)m * e.ldaux + n0;
      if (e.bias) {
#pragma unroll
        for (int j = 0; j < NV; j += 4) {
          float4 b = *reinterpret_cast<const float4*>(e.bias + n0 + j);
          v[j] += b.x; v[j + 1] += b.y; v[j + 2] += b.z; v[j + 3] += b.w;
        }
      }
#pragma unroll
      for (int j = 0; j < NV; j += 8) st_bf16x8(a + j, v + j);
      float gv[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) gv[j] = gelu_f(__bfloat162float(__float2bfloat16_rn(v[j])));
#pragma unroll
      for (int j = 0; j < NV; j += 8) st_bf16x8(c + j, gv + j);
    } break;
    case ADAPTRA_EPI_RESID: {
      bf16* c = (bf16*)e.C + (long)m * e.ldc + n0;
      const bf16* r = (const bf16*)e.R + (long)m * e.ldr + n0;
      float rv[NV];
#pragma unroll
      for (int j = 0; j < NV; j += 8) ld_bf16x8(r + j, rv + j);
      if (e.bias) {
#pragma unroll
        for (int j = 0; j < NV; j += 4) {
          float4 b = *reinterpret_cast<const float4*>(e.bias + n0 + j);
          v[j] += b.x; v[j + 1] += b.y; v[j + 2] += b.z; v[j + 3] += b.w;
        }
      }
#pragma unroll
      for (int j = 0; j < NV; ++j) v[j] += rv[j];
#pragma unroll
      for (int j = 0; j < NV; j += 8) st_bf16x8(c + j, v + j);
    } break;
    case ADAPTRA_EPI_DGELU: {
      bf16* c = (bf16*)e.C + (long)m * e.ldc + n0;
      const bf16* a = (const bf16*)e.aux + (long)m * e.ldaux + n0;
      float av[NV];
#pragma unroll
      for (int j = 0; j < NV; j += 8) ld_bf16x8(a + j, av + j);
#pragma unroll
      for (int j = 0; j < NV; ++j) v[j] *= gelu_grad_f(av[j]);
#pragma unroll
      for (int j = 0; j < NV; j += 8) st_bf16x8(c + j, v + j);
    } break;
    case ADAPTRA_EPI_ACC_F32: {
      float* c = (float*)e.C + (long)m * e.ldc + n0;
#pragma unroll
      for (int j = 0; j < NV; j += 4) {
        float4 o = *reinterpret_cast<float4*>(c + j);
        o.x += e.alpha * v[j]; o.y += e.alpha * v[j + 1]; o.z += e.alpha * v[j + 2]; o.w += e.alpha * v[j + 3];
        *reinterpret_cast<float4*>(c + j) = o;
      }
    } break;
    case ADAPTRA_EPI_STORE_F32: {
      float* c = (float*)e.C + (long)m * e.ldc + n0;
#pragma unroll
      for (int j = 0; j < NV; j += 4)
        *reinterpret_cast<float4*>(c + j) = make_float4(e.alpha * v[j], e.alpha * v[j + 1], e.alpha * v[j + 2],
                                                        e.alpha * v[j + 3]);
    } break;
    case ADAPTRA_EPI_DSOFTMAX: {
      bf16* c = (bf16*)e.C + (long)m * e.ldc + n0;
      const bf16* p = (const bf16*)e.aux + (long)m * e.ldaux + n0;
      float pv[NV];
#pragma unroll
      for (int j = 0; j < NV; j += 8) ld_bf16x8(p + j, pv + j);
      float D = e.rowv[m];
#pragma unroll
      for (int j = 0; j < NV; ++j) v[j] = pv[j] * (v[j] - D) * e.alpha;
#pragma unroll
      for (int j = 0; j < NV; j += 8) st_bf16x8(c + j, v + j);
    } break;
  }
}

__device__ __forceinline__ void epi_row32_bf16_fast(const EpiCtx& e, int m, int n0, float (&v)[32]) {
  epi_rowN_bf16_fast<32>(e, m, n0, v);
}

}  // namespace adaptra
