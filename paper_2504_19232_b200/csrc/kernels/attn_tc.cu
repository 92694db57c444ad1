// Fused causal attention on tcgen05 (bf16, head dim 128) for the GPT block of
// stage F / B: softmax(Q K^T / sqrt(dh)) V without materialising the
// T x T scores in HBM.
//
// Forward, one CTA per (sequence x head z, 128-query block qb):
//   pass 1: for key blocks j <= qb: S = Q K_j^T (TMEM) -> row max / sum
//   pass 2: for key blocks j <= qb: S = Q K_j^T -> P = exp(S/sqrt(dh) - LSE)
//           (bf16, shared memory) -> O += P V_j (TMEM)
//   O -> bf16 output, LSE = max + log(sum) (fp32, kept for B).
// Two passes trade one extra Q K^T per block for exact normalisation without
// rescaling the TMEM accumulator.
// Backward, one CTA per (z, 128-key block kb), over query blocks i >= kb:
//   S^T = K Q_i^T, dP^T = V dO_i^T (TMEM) -> P^T = exp(S^T/sqrt(dh) - LSE_i),
//   dS^T = P^T (dP^T - D_i) (bf16, shared memory) -> dV += P^T dO_i,
//   dK += dS^T Q_i, dQ_i(partial) = dS K (TMEM) -> TMA reduce-add into an fp32
//   dQ accumulator.  D_i = rowsum(dO_i o O_i) comes from attn_rowdot.
// Warp roles: 0 TMA producer, 1 TMEM allocator + MMA issuer, 2..5 softmax /
// gradient / epilogue warps (thread = TMEM lane = tile row).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>

#include "../../../include/adaptra.h"
#include "../prof.h"
#include "../util.h"
#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"

namespace adaptra {

namespace {
constexpr int AT = 128;        // rows per tile (queries or keys) and head dim
constexpr int CHUNK = 16384;   // one [128 rows x 64 cols] bf16 SWIZZLE_128B chunk
constexpr int TILE = 2 * CHUNK;  // [128 x 128] bf16 tile = 2 chunks
constexpr int kThreads = 192;

// K-major operand (rows x 128 cols in 2 chunks): k-step ks (16 columns)
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t base, int ks) {
  return umma_desc_sw128(base + (ks >> 2) * CHUNK + (ks & 3) * 32, 16, 1024);
}
// MN-major operand (128 K-rows x 128 MN in 2 chunks of 64): k-step ks = 16 rows
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t base, int ks) {
  return umma_desc_sw128(base + ks * 2048, CHUNK, 1024);
}
constexpr uint32_t idesc(int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(AT >> 3) << 17) | ((uint32_t)(AT >> 4) << 24);
}

// store 32 fp32 as bf16 into row r of a K-major SWIZZLE_128B [128 x 128] tile,
// columns [c0, c0 + 32)
__device__ __forceinline__ void st_tile_row32(uint8_t* tile, int r, int c0, const float* v) {
  uint8_t* chunk = tile + (c0 >> 6) * CHUNK + r * 128;
  const int p0 = (c0 & 63) >> 3;  // first 16-byte piece (8 columns) within the 128 B row
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u;
    u.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
    u.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
    u.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
    u.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
    *reinterpret_cast<uint4*>(chunk + (((p0 + q) ^ (r & 7)) << 4)) = u;
  }
}

struct AttnArgs {
  int b, H, T, d;        // sequences, heads, tokens per sequence, model width (= H * 128)
  float scale;           // 1 / sqrt(dh)
  // forward
  bf16* o;               // [b*T, d]
  float* lse;            // [b*H*T] log-sum-exp of the scaled scores, log2 units
  // backward
  const float* D;        // [b*H*T] rowsum(dO o O)
  bf16* dqkv;            // [b*T, 3d] (k and v sections written here)
  float* dq_acc;         // [b*T, d] fp32 accumulator of dQ (zeroed by the caller)
};
}  // namespace

// ============================================================== forward
constexpr int kAttnThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2..9 softmax
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// 1-D bulk copy global -> shared, completion counted on an mbarrier (16 B multiple)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQ = smem;                       // 32 KB
  uint8_t* sK = sQ + TILE;                  // 2 stages x 32 KB
  uint8_t* sV = sK + 2 * TILE;              // 2 stages x 32 KB
  uint8_t* sP = sV + 2 * TILE;              // 32 KB
  float* sStat = (float*)(sP + TILE);       // [2 halves][2 (m, l)][128]
  uint64_t* bar = (uint64_t*)(sStat + 4 * AT);
  uint64_t* q_full = bar + 0;
  uint64_t* kv_full = bar + 1;   // [2]
  uint64_t* kv_empty = bar + 3;  // [2]
  uint64_t* s_full = bar + 5;    // [2]
  uint64_t* s_empty = bar + 7;   // [2]
  uint64_t* p_full = bar + 9;
  uint64_t* p_empty = bar + 10;
  uint64_t* o_full = bar + 11;
  uint32_t* tmem_slot = (uint32_t*)(bar + 12);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nqb = a.T / AT, Z = a.b * a.H;
  const int qb = nqb - 1 - (int)(blockIdx.x / Z);  // heavy (late) query blocks first
  const int z = blockIdx.x % Z;
  const int s = z / a.H, h = z % a.H;
  const int row0 = s * a.T;                       // first row of this sequence in [b*T, .]
  const int qcol = h * AT, kcol = a.d + h * AT, vcol = 2 * a.d + h * AT;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 8);
    }
    mbar_init(p_full, 8);
    mbar_init(p_empty, 1);
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, TILE);
      for (int c = 0; c < 2; ++c) tma_load_2d(sQ + c * CHUNK, &tm_qkv, q_full, qcol + 64 * c, row0 + qb * AT);
      int st = 0;
      uint32_t ph = 0;
      for (int pass = 1; pass <= 2; ++pass) {
        for (int j = 0; j <= qb; ++j) {
          mbar_wait(&kv_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&kv_full[st], pass == 1 ? TILE : 2 * TILE);
          for (int c = 0; c < 2; ++c)
            tma_load_2d(sK + st * TILE + c * CHUNK, &tm_qkv, &kv_full[st], kcol + 64 * c, row0 + j * AT);
          if (pass == 2)
            for (int c = 0; c < 2; ++c)
              tma_load_2d(sV + st * TILE + c * CHUNK, &tm_qkv, &kv_full[st], vcol + 64 * c, row0 + j * AT);
          if (++st == 2) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // Block sequence g = 0..qb (pass 1), qb+1..2qb+1 (pass 2); K/V stage and S
    // buffer of block g are g & 1, their barrier phase (g >> 1) & 1.  In pass 2
    // S of block g+1 is issued before waiting for P of block g, so the softmax
    // warps overlap the tensor pipe.
    mbar_wait(q_full, 0);
    tc_fence_after();
    const uint32_t aQ = smem_u32(sQ), aP = smem_u32(sP);
    auto issue_s = [&](int gi) {
      const int st = gi & 1;
      const uint32_t ph = (gi >> 1) & 1;
      mbar_wait(&kv_full[st], ph);
      mbar_wait(&s_empty[st], ph ^ 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t aK = smem_u32(sK + st * TILE);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          tc_mma_f16(tmem + st * 128, desc_kmajor(aQ, ks), desc_kmajor(aK, ks), idesc(0, 0), ks > 0 ? 1u : 0u);
        tc_commit(&s_full[st]);
        if (gi <= qb) tc_commit(&kv_empty[st]);  // pass 1 only needs K
      }
      __syncwarp();
    };
    for (int gi = 0; gi <= qb; ++gi) issue_s(gi);
    const int g0 = qb + 1;
    issue_s(g0);
    for (int j = 0; j <= qb; ++j) {
      const int gi = g0 + j;
      if (j + 1 <= qb) issue_s(gi + 1);
      mbar_wait(p_full, j & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t aV = smem_u32(sV + (gi & 1) * TILE);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          tc_mma_f16(tO, desc_kmajor(aP, ks), desc_mnmajor(aV, ks), idesc(0, 1), (j > 0 || ks > 0) ? 1u : 0u);
        tc_commit(&kv_empty[gi & 1]);
        tc_commit(p_empty);
      }
      __syncwarp();
    }
    if (lane == 0) tc_commit(o_full);
    __syncwarp();
  } else {
    // softmax warps: lane quadrant quad (rows), column half (64 keys / head dims)
    const int quad = warp & 3, half = (warp - 2) >> 2;
    const int r = quad * 32 + lane;           // row within the query block
    const int qi = qb * AT + r;               // query position in the sequence
    const uint32_t lanes = ((uint32_t)(quad * 32) << 16) + half * 64;
    const float c2 = a.scale * kLog2e;        // scores in log2 units
    float m = -INFINITY, l = 0.f;
    // ---- pass 1: row max and sum (log2 domain) over this half of the keys
    for (int j = 0; j <= qb; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      uint32_t r0[32], r1[32];
      tmem_ld32(tmem + sb * 128 + lanes, r0);
      tmem_ld32(tmem + sb * 128 + lanes + 32, r1);
      tmem_ld_wait_regs(r0);
      tmem_ld_wait_regs(r1);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[sb]);
      float u[64];
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        u[t] = __uint_as_float(r0[t]) * c2;
        u[32 + t] = __uint_as_float(r1[t]) * c2;
      }
      if (j == qb) {
        const int key0 = j * AT + half * 64;
#pragma unroll
        for (int t = 0; t < 64; ++t)
          if (key0 + t > qi) u[t] = -INFINITY;
      }
      float cm = u[0];
#pragma unroll
      for (int t = 1; t < 64; ++t) cm = fmaxf(cm, u[t]);
      const float mn = fmaxf(m, cm);
      if (mn != -INFINITY) {
        float acc = 0.f;
#pragma unroll
        for (int t = 0; t < 64; ++t) acc += ex2(u[t] - mn);
        l = l * ex2(m - mn) + acc;
        m = mn;
      }
    }
    // combine the two halves of the row
    sStat[(half * 2 + 0) * AT + r] = m;
    sStat[(half * 2 + 1) * AT + r] = l;
    named_sync(1, 256);
    const float m0 = sStat[0 * AT + r], l0 = sStat[1 * AT + r];
    const float m1 = sStat[2 * AT + r], l1 = sStat[3 * AT + r];
    const float M = fmaxf(m0, m1);
    const float lse2 = M + __log2f(l0 * ex2(m0 - M) + l1 * ex2(m1 - M));
    // ---- pass 2: P = 2^(S c2 - lse2) -> shared memory
    for (int j = 0; j <= qb; ++j) {
      const int gi = qb + 1 + j, sb = gi & 1;
      mbar_wait(&s_full[sb], (gi >> 1) & 1);
      tc_fence_after();
      uint32_t r0[32], r1[32];
      tmem_ld32(tmem + sb * 128 + lanes, r0);
      tmem_ld32(tmem + sb * 128 + lanes + 32, r1);
      tmem_ld_wait_regs(r0);
      tmem_ld_wait_regs(r1);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[sb]);
      float p[64];
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        p[t] = ex2(fmaf(__uint_as_float(r0[t]), c2, -lse2));
        p[32 + t] = ex2(fmaf(__uint_as_float(r1[t]), c2, -lse2));
      }
      if (j == qb) {
        const int key0 = j * AT + half * 64;
#pragma unroll
        for (int t = 0; t < 64; ++t)
          if (key0 + t > qi) p[t] = 0.f;
      }
      mbar_wait(p_empty, (j & 1) ^ 1);  // previous P V has read the P buffer
      st_tile_row32(sP, r, half * 64, p);
      st_tile_row32(sP, r, half * 64 + 32, p + 32);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // ---- epilogue: O -> bf16 (this half of the head dims), LSE (log2 units)
    mbar_wait(o_full, 0);
    tc_fence_after();
    bf16* orow = a.o + (size_t)(row0 + qi) * a.d + h * AT + half * 64;
    uint32_t r0[32], r1[32];
    tmem_ld32(tO + lanes, r0);
    tmem_ld32(tO + lanes + 32, r1);
    tmem_ld_wait_regs(r0);
    tmem_ld_wait_regs(r1);
    float v[64];
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      v[t] = __uint_as_float(r0[t]);
      v[32 + t] = __uint_as_float(r1[t]);
    }
#pragma unroll
    for (int t = 0; t < 64; t += 8) st_bf16x8(orow + t, v + t);
    if (half == 0) a.lse[(size_t)z * a.T + qi] = lse2;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ============================================================== backward
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_dq, const AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sK = smem;            // 32 KB
  uint8_t* sV = sK + TILE;       // 32 KB
  uint8_t* sQ = sV + TILE;       // 32 KB (query block i)
  uint8_t* sdO = sQ + TILE;      // 32 KB
  uint8_t* sPT = sdO + TILE;     // 32 KB  P^T  [keys x queries]
  uint8_t* sdST = sPT + TILE;    // 32 KB  dS^T [keys x queries]
  uint8_t* sStg = sdST + TILE;   // 8 warps x 4 KB dQ staging
  float* sLse = (float*)(sStg + 8 * 4096);  // [128] (log2 units)
  float* sD = sLse + AT;                    // [128]
  uint64_t* bar = (uint64_t*)(sD + AT);
  uint64_t* kv_full = bar + 0;
  uint64_t* qd_full = bar + 1;
  uint64_t* qd_empty = bar + 2;
  uint64_t* sd_full = bar + 3;   // S^T and dP^T in TMEM
  uint64_t* pd_full = bar + 4;   // P^T, dS^T in smem (8 warps)
  uint64_t* pd_empty = bar + 5;  // MMAs done reading P^T, dS^T
  uint64_t* dq_full = bar + 6;   // dQ partial in TMEM
  uint64_t* dq_empty = bar + 7;  // dQ drained (8 warps)
  uint64_t* kv_done = bar + 8;   // dK, dV final
  uint32_t* tmem_slot = (uint32_t*)(bar + 9);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nb = a.T / AT, Z = a.b * a.H;
  const int kb = (int)(blockIdx.x / Z);  // heavy (early) key blocks first
  const int z = blockIdx.x % Z;
  const int s = z / a.H, h = z % a.H;
  const int row0 = s * a.T;
  const int qcol = h * AT, kcol = a.d + h * AT, vcol = 2 * a.d + h * AT;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_dq);
    mbar_init(kv_full, 1);
    mbar_init(qd_full, 1);
    mbar_init(qd_empty, 1);
    mbar_init(sd_full, 1);
    mbar_init(pd_full, 8);
    mbar_init(pd_empty, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 8);
    mbar_init(kv_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tdP = tmem + 128, tdV = tmem + 256, tdK = tmem + 384;
  const uint32_t tdQ = tmem;  // reuses the S^T columns once they are consumed

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * TILE);
      for (int c = 0; c < 2; ++c) {
        tma_load_2d(sK + c * CHUNK, &tm_qkv, kv_full, kcol + 64 * c, row0 + kb * AT);
        tma_load_2d(sV + c * CHUNK, &tm_qkv, kv_full, vcol + 64 * c, row0 + kb * AT);
      }
      uint32_t ph = 0;
      for (int i = kb; i < nb; ++i) {
        mbar_wait(qd_empty, ph ^ 1);
        mbar_arrive_expect_tx(qd_full, 2 * TILE + 2 * AT * 4);
        for (int c = 0; c < 2; ++c) {
          tma_load_2d(sQ + c * CHUNK, &tm_qkv, qd_full, qcol + 64 * c, row0 + i * AT);
          tma_load_2d(sdO + c * CHUNK, &tm_do, qd_full, h * AT + 64 * c, row0 + i * AT);
        }
        bulk_g2s(sLse, a.lse + (size_t)z * a.T + i * AT, AT * 4, qd_full);
        bulk_g2s(sD, a.D + (size_t)z * a.T + i * AT, AT * 4, qd_full);
        ph ^= 1;
      }
    }
  } else if (warp == 1) {
    mbar_wait(kv_full, 0);
    tc_fence_after();
    const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aQ = smem_u32(sQ), adO = smem_u32(sdO);
    const uint32_t aPT = smem_u32(sPT), adST = smem_u32(sdST);
    uint32_t ph = 0;
    for (int i = kb; i < nb; ++i) {
      mbar_wait(qd_full, ph);
      mbar_wait(dq_empty, ph ^ 1);  // S^T / dQ columns free
      tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          tc_mma_f16(tS, desc_kmajor(aK, ks), desc_kmajor(aQ, ks), idesc(0, 0), ks > 0 ? 1u : 0u);
          tc_mma_f16(tdP, desc_kmajor(aV, ks), desc_kmajor(adO, ks), idesc(0, 0), ks > 0 ? 1u : 0u);
        }
        tc_commit(sd_full);
      }
      __syncwarp();
      mbar_wait(pd_full, ph);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t acc = (i > kb) ? 1u : 0u;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)  // dQ_i = dS K first: its drain overlaps dV, dK
          tc_mma_f16(tdQ, desc_mnmajor(adST, ks), desc_mnmajor(aK, ks), idesc(1, 1), ks > 0 ? 1u : 0u);
        tc_commit(dq_full);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          // dV += P^T dO_i ; dK += dS^T Q_i  (B operands read MN-major)
          tc_mma_f16(tdV, desc_kmajor(aPT, ks), desc_mnmajor(adO, ks), idesc(0, 1), (acc || ks > 0) ? 1u : 0u);
          tc_mma_f16(tdK, desc_kmajor(adST, ks), desc_mnmajor(aQ, ks), idesc(0, 1), (acc || ks > 0) ? 1u : 0u);
        }
        tc_commit(pd_empty);
        tc_commit(qd_empty);
      }
      __syncwarp();
      ph ^= 1;
    }
    if (lane == 0) tc_commit(kv_done);
    __syncwarp();
  } else {
    const int quad = warp & 3, half = (warp - 2) >> 2;
    const int r = quad * 32 + lane;  // key row (S^T, dP^T, dK, dV) / query row (dQ)
    const int kj = kb * AT + r;      // key position
    const uint32_t lanes = ((uint32_t)(quad * 32) << 16) + half * 64;
    const float c2 = a.scale * kLog2e;
    uint8_t* stg = sStg + (warp - 2) * 4096;
    uint32_t ph = 0;
    for (int i = kb; i < nb; ++i) {
      mbar_wait(sd_full, ph);
      tc_fence_after();
      uint32_t rs0[32], rs1[32];
      tmem_ld32(tS + lanes, rs0);
      tmem_ld32(tS + lanes + 32, rs1);
      tmem_ld_wait_regs(rs0);
      tmem_ld_wait_regs(rs1);
      float p[64], ds[64];
      const int q0 = i * AT + half * 64;
      const float* lse = sLse + half * 64;
      const float* Dq = sD + half * 64;
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        p[t] = ex2(fmaf(__uint_as_float(rs0[t]), c2, -lse[t]));
        p[32 + t] = ex2(fmaf(__uint_as_float(rs1[t]), c2, -lse[32 + t]));
      }
      if (i == kb) {
#pragma unroll
        for (int t = 0; t < 64; ++t)
          if (q0 + t < kj) p[t] = 0.f;
      }
      tmem_ld32(tdP + lanes, rs0);
      tmem_ld32(tdP + lanes + 32, rs1);
      tmem_ld_wait_regs(rs0);
      tmem_ld_wait_regs(rs1);
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        ds[t] = p[t] * (__uint_as_float(rs0[t]) - Dq[t]);
        ds[32 + t] = p[32 + t] * (__uint_as_float(rs1[t]) - Dq[32 + t]);
      }
      mbar_wait(pd_empty, ph ^ 1);  // previous MMAs done reading P^T / dS^T
      st_tile_row32(sPT, r, half * 64, p);
      st_tile_row32(sPT, r, half * 64 + 32, p + 32);
      st_tile_row32(sdST, r, half * 64, ds);
      st_tile_row32(sdST, r, half * 64 + 32, ds + 32);
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(pd_full);
      // dQ partial (thread = query row, this half of the head dims) -> TMA reduce-add
      mbar_wait(dq_full, ph);
      tc_fence_after();
      uint32_t rq0[32], rq1[32];
      tmem_ld32(tdQ + lanes, rq0);
      tmem_ld32(tdQ + lanes + 32, rq1);
      tmem_ld_wait_regs(rq0);
      tmem_ld_wait_regs(rq1);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dq_empty);
      auto drain = [&](const uint32_t(&rq)[32], int c) {
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
        uint8_t* frow = stg + lane * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(frow + ((q ^ (lane & 7)) << 4)) =
              make_float4(__uint_as_float(rq[4 * q]) * a.scale, __uint_as_float(rq[4 * q + 1]) * a.scale,
                          __uint_as_float(rq[4 * q + 2]) * a.scale, __uint_as_float(rq[4 * q + 3]) * a.scale);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_reduce_add_2d(&tm_dq, stg, h * AT + half * 64 + c * 32, row0 + i * AT + quad * 32);
          bulk_commit();
        }
      };
      drain(rq0, 0);
      drain(rq1, 1);
      ph ^= 1;
    }
    if (lane == 0) bulk_wait<0>();
    // dK (scaled), dV -> bf16 into dqkv (k and v sections), thread = key row
    mbar_wait(kv_done, 0);
    tc_fence_after();
    for (int which = 0; which < 2; ++which) {
      const uint32_t tb = (which == 0 ? tdK : tdV) + lanes;
      bf16* out = a.dqkv + (size_t)(row0 + kj) * 3 * a.d + (which == 0 ? a.d : 2 * a.d) + h * AT + half * 64;
      const float sc = which == 0 ? a.scale : 1.f;
      uint32_t r0[32], r1[32];
      tmem_ld32(tb, r0);
      tmem_ld32(tb + 32, r1);
      tmem_ld_wait_regs(r0);
      tmem_ld_wait_regs(r1);
      float v[64];
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        v[t] = __uint_as_float(r0[t]) * sc;
        v[32 + t] = __uint_as_float(r1[t]) * sc;
      }
#pragma unroll
      for (int t = 0; t < 64; t += 8) st_bf16x8(out + t, v + t);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// dQ (fp32 accumulator) -> bf16 q section of dqkv; clears the accumulator.
// One thread per 8 consecutive elements of a row (32-bit index math, 16 B
// stores).
__global__ void __launch_bounds__(256) dq_finalize_kernel(float* __restrict__ acc, bf16* __restrict__ dqkv, int rows,
                                                          int d) {
  const int per_row = d / 8;
  const int n = rows * per_row;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int r = k / per_row, c = (k - r * per_row) * 8;
    float4* src = reinterpret_cast<float4*>(acc + (size_t)r * d + c);
    float4 v0 = src[0], v1 = src[1];
    src[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    src[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    uint4 u;
    u.x = pack_bf16x2(v0.x, v0.y);
    u.y = pack_bf16x2(v0.z, v0.w);
    u.z = pack_bf16x2(v1.x, v1.y);
    u.w = pack_bf16x2(v1.z, v1.w);
    *reinterpret_cast<uint4*>(dqkv + (size_t)r * 3 * d + c) = u;
  }
}

// ============================================================== host
typedef CUresult (*PFN_encodeTiled2)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static int map2d(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld_elems, int esz,
                 int box_c, int box_r, CUtensorMapSwizzle swz) {
  static PFN_encodeTiled2 enc = nullptr;
  if (!enc) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return set_error(ADAPTRA_ECUDA, "cuTensorMapEncodeTiled unavailable");
    enc = (PFN_encodeTiled2)p;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld_elems * esz)};
  cuuint32_t box[2] = {(cuuint32_t)box_c, (cuuint32_t)box_r};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(ADAPTRA_ECUDA, "cuTensorMapEncodeTiled (attn) failed");
  return ADAPTRA_OK;
}

static int check_launch(const char* w) {
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ADAPTRA_ECUDA, std::string(w) + ": " + cudaGetErrorString(e));
  return ADAPTRA_OK;
}

constexpr int kFwdSmem = 6 * TILE + 4 * AT * 4 + 1024 + 256;
constexpr int kBwdSmem = 6 * TILE + 8 * 4096 + 2 * AT * 4 + 1024 + 256;

int attn_fwd_tc(const bf16* qkv, bf16* o, float* lse, int b, int H, int T, int d, cudaStream_t st) {
  if (d != H * AT || T % AT) return set_error(ADAPTRA_EINVAL, "attn_fwd_tc: head dim 128 and T % 128 required");
  CUtensorMap m;
  int rc = map2d(&m, qkv, (int64_t)b * T, 3LL * d, 3LL * d, 2, 64, AT, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  static unsigned attr = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr & (1u << dev))) {
    cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem);
    attr |= 1u << dev;
  }
  AttnArgs a{};
  a.b = b; a.H = H; a.T = T; a.d = d;
  a.scale = 1.f / std::sqrt((float)AT);
  a.o = o;
  a.lse = lse;
  void* pb = prof_on() ? prof_begin(st) : nullptr;
  attn_fwd_kernel<<<b * H * (T / AT), kAttnThreads, kFwdSmem, st>>>(m, a);
  if (pb) {
    double fl = 4.0 * (double)T * T * AT * b * H * 0.5;  // algorithmic: QK^T + PV, causal half (R28)
    prof_end(pb, st, PROF_ATTN, fl, 0);
  }
  return check_launch("attn_fwd_tc");
}

int attn_bwd_tc(const bf16* qkv, const bf16* dO, const float* lse, const float* D, bf16* dqkv, float* dq_acc, int b,
                int H, int T, int d, cudaStream_t st) {
  if (d != H * AT || T % AT) return set_error(ADAPTRA_EINVAL, "attn_bwd_tc: head dim 128 and T % 128 required");
  CUtensorMap mq, mdo, mdq;
  int rc = map2d(&mq, qkv, (int64_t)b * T, 3LL * d, 3LL * d, 2, 64, AT, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = map2d(&mdo, dO, (int64_t)b * T, d, d, 2, 64, AT, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = map2d(&mdq, dq_acc, (int64_t)b * T, d, d, 4, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  static unsigned attr = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr & (1u << dev))) {
    cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdSmem);
    attr |= 1u << dev;
  }
  AttnArgs a{};
  a.b = b; a.H = H; a.T = T; a.d = d;
  a.scale = 1.f / std::sqrt((float)AT);
  a.lse = const_cast<float*>(lse);
  a.D = D;
  a.dqkv = dqkv;
  a.dq_acc = dq_acc;
  void* pb = prof_on() ? prof_begin(st) : nullptr;
  attn_bwd_kernel<<<b * H * (T / AT), kAttnThreads, kBwdSmem, st>>>(mq, mdo, mdq, a);
  if (pb) {
    double fl = 8.0 * (double)T * T * AT * b * H * 0.5;  // dP, dV, dK, dQ (causal half)
    prof_end(pb, st, PROF_ATTN, fl, 0);
  }
  rc = check_launch("attn_bwd_tc");
  if (rc) return rc;
  const int n8 = b * T * (d / 8);
  dq_finalize_kernel<<<std::min(148 * 8, (n8 + 255) / 256), 256, 0, st>>>(dq_acc, dqkv, b * T, d);
  return check_launch("dq_finalize");
}

}  // namespace adaptra
