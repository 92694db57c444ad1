// Fused causal attention on tcgen05 (bf16, head dim 128) for the GPT block of
// stage F / B: softmax(Q K^T / sqrt(dh)) V without materialising the
// T x T scores in HBM.
//
// Forward, one CTA per (sequence x head z, 128-query block qb), one pass over
// key blocks j <= qb: S = Q K_j^T (TMEM) -> online softmax against a lazily
// moved reference max (P = 2^(S c2 - mref) <= 2^8, bf16, shared memory;
// O rescaled in TMEM only when mref moves) -> O += P V_j (TMEM);
// O / l -> bf16 output, LSE = mref + log2(l) (log2 units, kept for B).
// Backward, one CTA per (z, 128-key block kb), over 64-query blocks i >= 2 kb:
//   S^T = K Q_i^T, dP^T = V dO_i^T (TMEM) -> P^T = exp(S^T/sqrt(dh) - LSE_i),
//   dS^T = P^T (dP^T - D_i) (bf16, shared memory) -> dV += P^T dO_i,
//   dK += dS^T Q_i, dQ_i^T(partial) = K^T dS_i^T (TMEM) -> TMA reduce-add into
//   an fp32 dQ^T accumulator.  D_i = rowsum(dO_i o O_i) comes from the epilogue
//   of the GEMM that produces dO (EPI_STORE_ROWDOT; attn_rowdot elsewhere).
// Warp roles: 0 TMA producer, 1 TMEM allocator + MMA issuer; forward: 2..9
// (or 2..17) softmax / epilogue warps (lane quadrant x column group); backward: 2..17
// gradient warps (lane quadrant x 16-query column group), 18..21 dQ^T drain
// warps (thread = TMEM lane = tile row).
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

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

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
// store 32 fp32 as bf16 into row r of a K-major SWIZZLE_128B [128 x 128] tile
// (shared address `tile`), columns [c0, c0 + 32)
__device__ __forceinline__ void st_tile_row32(uint32_t tile, int r, int c0, const float* v) {
  const uint32_t row = tile + (c0 >> 6) * CHUNK + r * 128;
  const int p0 = (c0 & 63) >> 3;  // first 16-byte piece (8 columns) within the 128 B row
#pragma unroll
  for (int q = 0; q < 4; ++q)
    sts128(row + (((p0 + q) ^ (r & 7)) << 4), pack_bf16x2(v[8 * q + 0], v[8 * q + 1]),
           pack_bf16x2(v[8 * q + 2], v[8 * q + 3]), pack_bf16x2(v[8 * q + 4], v[8 * q + 5]),
           pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
}
// same, from 32 values already packed as 16 bf16x2 words
__device__ __forceinline__ void st_tile_row32_packed(uint32_t tile, int r, int c0, const uint32_t* pk) {
  const uint32_t row = tile + (c0 >> 6) * CHUNK + r * 128;
  const int p0 = (c0 & 63) >> 3;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    sts128(row + (((p0 + q) ^ (r & 7)) << 4), pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
}

// wait for this thread's outstanding tcgen05.ld into r[0..N) (N multiple of 32)
template <int N>
__device__ __forceinline__ void tmem_ld_wait_regs_n(uint32_t (&r)[N]) {
#pragma unroll
  for (int c = 0; c < N / 32; ++c) tmem_ld_wait_regs(*reinterpret_cast<uint32_t(*)[32]>(&r[32 * c]));
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
  long long* trace;      // diag 0x200: per-iteration clock64 stamps of CTA 0 ([it][16])
  long long* cta;        // diag 0x400: per CTA {smid, globaltimer at entry, at exit}
  int diag;              // ADAPTRA_ATTN_DIAG bit mask, timing experiments only (0 = normal): 1 no dQ
                         // reduce, 2 no gradient math, 4 no MMAs, 8 no Q/dO loads, 0x10/0x20/0x40/0x80/0x100 no S/dP/dV/dK/dQ MMA
};
}  // namespace

// ============================================================== forward
// Softmax warps: NQ per TMEM lane quadrant, each owning 128 / NQ of a row's
// 128 columns (NQ = 2: 8 warps, 64 columns per thread; NQ = 4: 16 warps, 32
// columns, 4 warps per SM sub-partition; $ADAPTRA_ATTN_FWD_WARPS = 8 | 16).
template <int NQ>
struct FwdCfg {
  static constexpr int kSoftWarps = 4 * NQ;
  static constexpr int kThreads = 64 + 32 * kSoftWarps;  // warp 0 TMA, warp 1 MMA, then softmax
  static constexpr int kRing = NQ == 2 ? 5 : 4;         // K/V tile ring (2.5 / 2 key blocks of TMA lead)
  static constexpr int kCols = 128 / NQ;                 // columns per softmax thread
  static constexpr int kSmem = (kRing + 2) * TILE + 2 * NQ * AT * 4 + 256;
};
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int smid() {
  int v;
  asm volatile("mov.u32 %0, %smid;" : "=r"(v));
  return v;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA / ALU pipes, to take part of the softmax off the MUFU unit
// (16 ex2 per clock per SM): x = j + f with j = rint(x) (the 1.5 * 2^23
// round-to-integer trick; j lands in t's low mantissa bits), 2^f on
// [-0.5, 0.5] by a degree-3 polynomial (relative error 7.5e-5, below the
// 2^-9 of the bf16 P it feeds), 2^j added into the exponent field.  x is
// clamped at -126 (masked keys, -inf, give ~2^-126 instead of 0).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = __fadd_rn(x, 12582912.f);
  const float f = __fsub_rn(x, __fsub_rn(t, 12582912.f));
  float p = fmaf(0.0551716648f, f, 0.2426111251f);
  p = fmaf(p, f, 0.6932609677f);
  p = fmaf(p, f, 0.9999280572f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// 1-D bulk copy global -> shared, completion counted on an mbarrier (16 B multiple)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Persistent: one CTA per SM walks work items (z, qb) -- heavy (late) query
// blocks first, dealt to the CTAs in snake order (round r: item r*G + c, then
// (r+1)*G - 1 - c), so each SM's total key blocks stay close to the mean.  The
// K/V ring, the S buffers and every barrier phase run on counters global to
// the CTA, so the next item's Q / K / V loads and its first S MMA overlap this
// item's last softmax block and epilogue (per-CTA setup and the epilogue were
// 26 % of the SM time with one CTA per item, diag 0x400).
__device__ __forceinline__ int fwd_item(int r, int c, int G) { return (r & 1) ? (r + 1) * G - 1 - c : r * G + c; }

// POLY of every 4 exponentials per thread go through ex2_poly ($ADAPTRA_ATTN_POLY).
// PT = 1: P stays in TMEM -- written as bf16 pairs over the S columns each
// thread has read (k-step ks of P V reads columns [16 ks, 16 ks + 8) of the S
// buffer) and consumed as the A operand of P V from there (the ts form): the
// M = 128 MMAs no longer read P from shared memory (and nothing writes it
// there), which with Q, K, V and the TMA fills is the shared-memory traffic
// that bounds the block.  The S buffer is then released by P V's commit.
// QT = 1 (with PT): Q moves to TMEM too (columns [384, 512): two 64-column
// buffers, one per item parity) and S = Q K^T runs in the ts form, so the
// S MMAs read only K from shared memory.  Four more warps copy each item's Q
// from its TMA tile into TMEM (thread = query row) once the item two back has
// issued its last S; the Q tile in shared memory is free right after.
// S2 = 1 (with PT = 1, three S buffers): the S products are issued by a warp
// of their own (warp 2 + kSoftWarps), so S(g + 1) no longer waits in one
// issue stream behind P V(g - 1); each issuer commits its own MMAs.
template <int NQ, int POLY, int PT = 0, int QT = 0, int S2 = 0>
__global__ void __launch_bounds__(FwdCfg<NQ>::kThreads + (QT ? 128 : 0) + (S2 ? 32 : 0), 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const AttnArgs a) {
  constexpr int kFwdRing = FwdCfg<NQ>::kRing, kSoftWarps = FwdCfg<NQ>::kSoftWarps, CW = FwdCfg<NQ>::kCols;
  // S buffers in TMEM: with P in TMEM a buffer is busy until its P V is done,
  // so S(g + 1) with two buffers would wait for P V(g - 1) to drain the tensor
  // pipe; three keep it fed (O then sits at column 384; QT needs 384+ for Q)
  // PT = 2 (with QT): one S buffer, released as soon as the softmax has
  // loaded it, and P in two separate 64-column buffers -- S(g + 1) then
  // overlaps the softmax of block g, S reads only K from shared memory (Q
  // is in TMEM) and nothing waits for a P V to drain.  TMEM: S [0, 128),
  // O [128, 256), P [256, 384), Q [384, 512).
  constexpr bool SEP = PT == 2;
  static_assert(!SEP || QT, "PT = 2 needs Q in TMEM");
  constexpr int NS = SEP ? 1 : ((PT && !QT) ? 3 : 2);
  static_assert(!S2 || (PT == 1 && !QT), "S2 needs P in TMEM with three S buffers");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;  // no static shared memory: the window starts 1024-aligned (checked)
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023)) __trap();
  uint8_t* sQ = smem;                       // 32 KB
  uint8_t* sRing = sQ + TILE;               // kFwdRing x 32 KB: K V K V ... (tile n in slot n % kFwdRing)
  uint8_t* sP = sRing + kFwdRing * TILE;    // 32 KB
  float* sMax = (float*)(sP + TILE);        // [2 (block parity)][NQ column groups][128] partial row maxima
  uint64_t* bar = (uint64_t*)(sMax + 2 * NQ * AT);
  uint64_t* q_full = bar + 0;
  uint64_t* t_full = bar + 1;               // [kFwdRing] tile landed
  uint64_t* t_empty = t_full + kFwdRing;    // [kFwdRing] tile consumed by its MMA
  uint64_t* s_full = t_empty + kFwdRing;    // [NS]
  uint64_t* s_empty = s_full + NS;          // [NS]
  uint64_t* p_full = s_empty + NS;
  uint64_t* p_empty = p_full + 1;           // [2] (SEP: per P buffer; else [0] only)
  uint64_t* o_full = p_empty + 2;
  uint64_t* q_empty = o_full + 1;           // the item's last S MMA read Q (QT: the copy warps read it)
  uint64_t* qt_full = q_empty + 1;          // QT: [2] Q of the item in TMEM buffer it & 1
  uint64_t* qt_empty = qt_full + 2;         // QT: [2] that item's last S MMA done
  uint32_t* tmem_slot = (uint32_t*)(qt_empty + 2);

  const long long cta_t0 = (a.diag & 0x400) ? gtimer() : 0;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nqb = a.T / AT, Z = a.b * a.H, n_items = nqb * Z;
  const int G = (int)gridDim.x, cta = (int)blockIdx.x;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    mbar_init(q_full, 1);
    mbar_init(q_empty, QT ? 4 : 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&qt_full[i], 4);
      mbar_init(&qt_empty[i], 1);
    }
    for (int i = 0; i < kFwdRing; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], 1);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], PT == 1 ? 1 : kSoftWarps);
    }
    mbar_init(p_full, kSoftWarps);
    mbar_init(&p_empty[0], 1);
    mbar_init(&p_empty[1], 1);
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem + (SEP ? 128 : NS * 128);

  if (warp == 0) {
    if (lane == 0) {
      int slot = 0, ph = 0;
      for (int r = 0, it = 0;; ++r, ++it) {
        const int item = fwd_item(r, cta, G);
        if (item >= n_items) break;
        const int qb = nqb - 1 - item / Z, z = item % Z;
        const int s = z / a.H, h = z % a.H, row0 = s * a.T;
        const int kcol = a.d + h * AT, vcol = 2 * a.d + h * AT;
        mbar_wait(q_empty, (it & 1) ^ 1);
        mbar_arrive_expect_tx(q_full, TILE);
        for (int c = 0; c < 2; ++c) tma_load_2d(sQ + c * CHUNK, &tm_qkv, q_full, h * AT + 64 * c, row0 + qb * AT);
        for (int n = 0; n < 2 * (qb + 1); ++n) {  // K_j (n = 2j), V_j (n = 2j+1)
          mbar_wait(&t_empty[slot], ph ^ 1);
          mbar_arrive_expect_tx(&t_full[slot], TILE);
          const int col = (n & 1) ? vcol : kcol;
          for (int c = 0; c < 2; ++c)
            tma_load_2d(sRing + slot * TILE + c * CHUNK, &tm_qkv, &t_full[slot], col + 64 * c, row0 + (n >> 1) * AT);
          if (++slot == kFwdRing) {
            slot = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1 || (S2 && warp == 2 + kSoftWarps)) {
    // S2: warp 1 issues the P V products, warp 2 + kSoftWarps the S products
    const bool do_s = !S2 || warp != 1, do_pv = !S2 || warp == 1;
    // S of block j+1 is issued before waiting for P of block j, so the softmax
    // warps overlap the tensor pipe; across items, S of the next item's first
    // block follows this item's last P V.  Global block g: S buffer
    // g % NS, K tile 2g and V tile 2g+1 of the ring.
    const uint32_t aQ = smem_u32(sQ), aP = smem_u32(sP);
    // S of global block g; QT: Q from TMEM buffer qb
    auto issue_s = [&](int g, int qb) {
      const int st = g % NS;
      const int slot = (2 * g) % kFwdRing;
      mbar_wait(&t_full[slot], ((2 * g) / kFwdRing) & 1);
      mbar_wait(&s_empty[st], ((g / NS) & 1) ^ 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t aK = smem_u32(sRing + slot * TILE);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          if (QT)
            tc_mma_f16_ts(tmem + st * 128, tmem + 384 + qb * 64 + 8 * ks, desc_kmajor(aK, ks), idesc(0, 0),
                          ks > 0 ? 1u : 0u);
          else
            tc_mma_f16(tmem + st * 128, desc_kmajor(aQ, ks), desc_kmajor(aK, ks), idesc(0, 0), ks > 0 ? 1u : 0u);
        }
        tc_commit(&s_full[st]);
        tc_commit(&t_empty[slot]);
      }
      __syncwarp();
    };
    // the item's Q is ready for its S MMAs
    auto wait_q = [&](int it) {
      if (QT)
        mbar_wait(&qt_full[it & 1], (it >> 1) & 1);
      else
        mbar_wait(q_full, it & 1);
      tc_fence_after();
    };
    int g0 = 0;  // global index of the item's first block
    int it = 0;
    int item = fwd_item(0, cta, G);
    if (item < n_items && do_s) {
      wait_q(0);
      issue_s(0, 0);
    }
    // diag 0x200: clock64 stamps of CTA 0's first 64 blocks ([g][16]): 0 S(g+1)
    // issued, 1 P(g) seen, 2 P V(g) issued; softmax warp 2: 3 S(g) seen, 4 S
    // loaded, 5 row max exchanged, 6 exponentials done, 7 O ready, 8 P written
    const bool trm = (a.diag & 0x200) && blockIdx.x == 0 && lane == 0;
#define FTRACE(on, g, ev) \
  if ((on) && (g) < 64) a.trace[(g) * 16 + (ev)] = clock64();
    while (item < n_items) {
      const int nb = nqb - item / Z;  // key blocks of this item
      const int next = fwd_item(it + 1, cta, G);
      for (int j = 0; j < nb; ++j) {
        const int g = g0 + j;
        if (!do_s) {
        } else if (j + 1 < nb) {
          issue_s(g + 1, it & 1);
          FTRACE(trm, g, 0)
        } else {
          // after the item's last S: Q may be replaced
          if (lane == 0) tc_commit(QT ? &qt_empty[it & 1] : q_empty);
          __syncwarp();
        }
        if (!do_pv) continue;
        const int vslot = (2 * g + 1) % kFwdRing;
        mbar_wait(p_full, g & 1);
        FTRACE(trm, g, 1)
        mbar_wait(&t_full[vslot], ((2 * g + 1) / kFwdRing) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t aV = smem_u32(sRing + vslot * TILE);
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            if (SEP)
              tc_mma_f16_ts(tO, tmem + 256 + (g & 1) * 64 + 8 * ks, desc_mnmajor(aV, ks), idesc(0, 1),
                            (j > 0 || ks > 0) ? 1u : 0u);
            else if (PT)
              tc_mma_f16_ts(tO, tmem + (g % NS) * 128 + 16 * ks, desc_mnmajor(aV, ks), idesc(0, 1),
                            (j > 0 || ks > 0) ? 1u : 0u);
            else
              tc_mma_f16(tO, desc_kmajor(aP, ks), desc_mnmajor(aV, ks), idesc(0, 1), (j > 0 || ks > 0) ? 1u : 0u);
          }
          tc_commit(&t_empty[vslot]);
          tc_commit(&p_empty[SEP ? (g & 1) : 0]);
          if (PT == 1) tc_commit(&s_empty[g % NS]);  // P (in the S buffer) consumed
        }
        FTRACE(trm, g, 2)
        __syncwarp();
      }
      if (do_pv && lane == 0) tc_commit(o_full);
      __syncwarp();
      // the next item's first S: its Q load started when this item's last S
      // finished, so it lands while the softmax warps run the last block and
      // the epilogue (waiting here before the last P V would put it on the path)
      if (next < n_items && do_s) {
        wait_q(it + 1);
        issue_s(g0 + nb, (it + 1) & 1);
      }
      g0 += nb;
      ++it;
      item = next;
    }
  } else if (QT && warp >= 2 + kSoftWarps) {
    // Q copy warps (QT): thread = query row r; its two 128-byte rows of the
    // K-major SWIZZLE_128B Q tile (logical 16-byte piece p at p ^ (r & 7))
    // become 64 TMEM columns of bf16 pairs, the A layout of the ts-form S MMA
    const int quad = warp & 3, r = quad * 32 + lane;
    const uint32_t lanes = (uint32_t)(quad * 32) << 16;
    for (int rr = 0, it = 0;; ++rr, ++it) {
      if (fwd_item(rr, cta, G) >= n_items) break;
      const int b = it & 1;
      mbar_wait(q_full, it & 1);
      mbar_wait(&qt_empty[b], ((it >> 1) & 1) ^ 1);  // item it - 2's last S done with this buffer
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t w[32];
        const uint32_t row = smem_u32(sQ) + c * CHUNK + r * 128;
#pragma unroll
        for (int p = 0; p < 8; ++p)
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(w[4 * p]), "=r"(w[4 * p + 1]), "=r"(w[4 * p + 2]), "=r"(w[4 * p + 3])
                       : "r"(row + ((p ^ (r & 7)) << 4)));
        tmem_st32(tmem + 384 + b * 64 + lanes + 32 * c, w);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&qt_full[b]);
        mbar_arrive(q_empty);  // the Q tile in shared memory is free
      }
    }
  } else {
    // softmax warps: lane quadrant quad (rows), column group qtr (CW keys /
    // head dims).  Online softmax in log2 units against a reference max mref
    // shared by the NQ groups of a row (exchanged through sMax every block).
    // mref moves only when the running max exceeds it by more than 8, so
    // P <= 2^8 and the O accumulator in TMEM is rescaled rarely (then by this
    // thread's group).  The next item's first P V (which overwrites O) waits
    // for p_full, which these warps arrive only after reading O in the epilogue.
    const int quad = warp & 3, qtr = (warp - 2) >> 2;
    const int r = quad * 32 + lane;           // row within the query block
    const uint32_t lanes = ((uint32_t)(quad * 32) << 16) + qtr * CW;
    const float c2 = a.scale * kLog2e;        // scores in log2 units
    const int row_bar = 1 + quad;             // the NQ warps of lane quadrant quad
    int g = 0;
    for (int rr = 0, it = 0;; ++rr, ++it) {
      const int item = fwd_item(rr, cta, G);
      if (item >= n_items) break;
      const int qb = nqb - 1 - item / Z, z = item % Z;
      const int s = z / a.H, h = z % a.H, row0 = s * a.T;
      const int qi = qb * AT + r;             // query position in the sequence
      float mref = -INFINITY, l = 0.f;
      for (int j = 0; j <= qb; ++j, ++g) {
        const int sb = g & 1;   // row-max exchange parity
        const int tb = g % NS;  // TMEM S buffer
        const bool trs = (a.diag & 0x200) && blockIdx.x == 0 && warp == 2 && lane == 0;
        mbar_wait(&s_full[tb], (g / NS) & 1);
        FTRACE(trs, g, 3)
        tc_fence_after();
        uint32_t rv[CW];
#pragma unroll
        for (int c = 0; c < CW / 32; ++c) tmem_ld32(tmem + tb * 128 + lanes + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&rv[32 * c]));
        tmem_ld_wait_regs_n<CW>(rv);
        FTRACE(trs, g, 4)
        tc_fence_before();
        __syncwarp();
        if (PT != 1 && lane == 0) mbar_arrive(&s_empty[tb]);
        if (j == qb) {
          const int lim = qi - (j * AT + qtr * CW);  // last visible column of this group
#pragma unroll
          for (int t = 0; t < CW; ++t)
            if (t > lim) rv[t] = __float_as_uint(-INFINITY);
        }
        float cm = __uint_as_float(rv[0]);
#pragma unroll
        for (int t = 1; t < CW; ++t) cm = fmaxf(cm, __uint_as_float(rv[t]));
        float* mx = sMax + sb * NQ * AT;
        mx[qtr * AT + r] = cm;
        named_sync(row_bar, 32 * NQ);
        // every row has key 0 <= qi in block 0 and key j*128 <= qi in block j: mb is finite
        float mall = mx[r];
#pragma unroll
        for (int k = 1; k < NQ; ++k) mall = fmaxf(mall, mx[k * AT + r]);
        const float mb = mall * c2;
        FTRACE(trs, g, 5)
        const bool resc = mb > mref + 8.f;
        float alpha = 1.f;
        if (resc) {
          alpha = ex2(mref - mb);  // 0 on the first block
          mref = mb;
        }
        uint32_t pk[CW / 2];  // P row group as bf16x2
        float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
        for (int t = 0; t < CW; t += 4) {
          const float e0 = ex2(fmaf(__uint_as_float(rv[t]), c2, -mref));
          const float e1 = ex2(fmaf(__uint_as_float(rv[t + 1]), c2, -mref));
          const float x2 = fmaf(__uint_as_float(rv[t + 2]), c2, -mref);
          const float x3 = fmaf(__uint_as_float(rv[t + 3]), c2, -mref);
          const float e2 = POLY >= 2 ? ex2_poly(x2) : ex2(x2);
          const float e3 = POLY >= 1 ? ex2_poly(x3) : ex2(x3);
          acc0 += e0 + e1;
          acc1 += e2 + e3;
          pk[t >> 1] = pack_bf16x2(e0, e1);
          pk[(t >> 1) + 1] = pack_bf16x2(e2, e3);
        }
        l = l * alpha + (acc0 + acc1);
        FTRACE(trs, g, 6)
        // P V of the previous block done before P(g) is written: O stable for
        // a rescale (and, without PT, the P buffer free).  The wait is kept
        // even when nothing is rescaled: P V(g - 1) needs every softmax warp's
        // p_full arrival for g - 1, so no warp can arrive for block g while
        // another has yet to arrive for g - 1 -- without it a fast warp's
        // arrival counted toward the previous phase of p_full (a P V on an
        // incomplete P, then an aliased parity: the intermittent 8-stage hang
        // of profiles/r02_attn_ptmem_hang.txt).
        const bool resc_o = j > 0 && __any_sync(0xffffffffu, resc);
        if (SEP) {
          if (g > 0) mbar_wait(&p_empty[(g - 1) & 1], ((g - 1) >> 1) & 1);
        } else if (PT == 1 && NS == 3) {
          // P V(g - 1) done = use (g - 1) / 3 of S buffer (g - 1) % 3 released
          // (a parity wait on the single p_empty could alias: with three S
          // buffers P V(g - 2) may still be running here)
          if (g > 0) mbar_wait(&s_empty[(g - 1) % NS], ((g - 1) / NS) & 1);
        } else {
          mbar_wait(&p_empty[0], (g & 1) ^ 1);
        }
        if (resc_o) {
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < CW / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(tO + lanes + 32 * c, o);
            tmem_ld_wait_regs(o);
#pragma unroll
            for (int t = 0; t < 32; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * alpha);
            tmem_st32(tO + lanes + 32 * c, o);
          }
          tmem_st_wait();
        }
        FTRACE(trs, g, 7)
        if (SEP) {
          // P buffer g & 1: P V(g - 2) has finished reading it; k-step ks of
          // this thread's keys at columns [8 ks, 8 ks + 8)
          mbar_wait(&p_empty[g & 1], ((g >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t pb = tmem + 256 + (g & 1) * 64 + ((uint32_t)(quad * 32) << 16) + qtr * (CW / 2);
#pragma unroll
          for (int c = 0; c < CW / 16; ++c) tmem_st8(pb + 8 * c, pk + 8 * c);
          tmem_st_wait();
        } else if (PT) {
#pragma unroll
          for (int c = 0; c < CW / 16; ++c) tmem_st8(tmem + tb * 128 + lanes + 16 * c, pk + 8 * c);
          tmem_st_wait();
        } else {
#pragma unroll
          for (int c = 0; c < CW / 32; ++c) st_tile_row32_packed(smem_u32(sP), r, qtr * CW + 32 * c, pk + 16 * c);
          fence_proxy_async_smem();
        }
        tc_fence_before();
        __syncwarp();
        FTRACE(trs, g, 8)
        if (lane == 0) mbar_arrive(p_full);
      }
      // ---- epilogue: O / l -> bf16 (this group of the head dims), LSE (log2
      // units).  The row sums are exchanged through the sMax buffer of the
      // parity the last block did not use (all groups finished reading it
      // before the last block's barrier); the second barrier keeps the next
      // item's first block, which writes that buffer, behind all reads.
      float* sL = sMax + (g & 1) * NQ * AT;
      sL[qtr * AT + r] = l;
      named_sync(row_bar, 32 * NQ);
      float ltot = 0.f;
#pragma unroll
      for (int k = 0; k < NQ; ++k) ltot += sL[k * AT + r];
      named_sync(row_bar, 32 * NQ);
      const float inv = 1.f / ltot;
      mbar_wait(o_full, it & 1);
      tc_fence_after();
      uint32_t rv[CW];
#pragma unroll
      for (int c = 0; c < CW / 32; ++c) tmem_ld32(tO + lanes + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&rv[32 * c]));
      tmem_ld_wait_regs_n<CW>(rv);
      tc_fence_before();
      bf16* orow = a.o + (size_t)(row0 + qi) * a.d + h * AT + qtr * CW;
      float v[CW];
#pragma unroll
      for (int t = 0; t < CW; ++t) v[t] = __uint_as_float(rv[t]) * inv;
#pragma unroll
      for (int t = 0; t < CW; t += 8) st_bf16x8(orow + t, v + t);
      if (qtr == 0) a.lse[(size_t)z * a.T + qi] = mref + __log2f(ltot);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
  if ((a.diag & 0x400) && threadIdx.x == 0) {
    a.cta[3 * blockIdx.x] = smid();
    a.cta[3 * blockIdx.x + 1] = cta_t0;
    a.cta[3 * blockIdx.x + 2] = gtimer();
  }
}

#undef FTRACE
// ============================================================== forward, ping-pong
// Two query tiles per work item -- blocks 2p (A) and 2p+1 (B) of one
// (sequence, head) -- share every K_j / V_j tile, and the tensor pipe
// alternates between them: S_A(j) = Q_A K_j^T, S_B(j), then O_A += P_A(j) V_j
// as soon as A's softmax warps have written P_A(j), S_A(j+1), O_B += P_B(j)
// V_j, S_B(j+1), ...  While one tile's softmax runs, the pipe works on the
// other's products, so softmax and MMA overlap instead of alternating.
// P is written back into the S columns of TMEM as bf16 pairs (16 keys per
// 8 columns) and consumed from there as the A operand of P V (the ts form),
// so it never touches shared memory.  TMEM: S_A [0,128), S_B [128,256),
// O_A [256,384), O_B [384,512).  Warps: 0 TMA, 1 MMA, 2..9 softmax of A,
// 10..17 softmax of B (lane quadrant x column half, as attn_fwd_kernel<2>).
// The same online softmax (lazy reference max, P <= 2^8), masking and
// epilogue as attn_fwd_kernel; one S buffer per tile: S_t(j+1) is issued only
// after P_t(j) V_j, which it overwrites, in the in-order tensor pipe.
constexpr int kPPThreads = 64 + 32 * 16;
constexpr int kPPRing = 4;
constexpr int kPPSmem = (2 + kPPRing) * TILE + 2 * 2 * 2 * AT * 4 + 256;
static_assert(kPPSmem <= 232448, "attn fwd ping-pong shared memory");

__device__ __forceinline__ int pp_item(int r, int c, int G) { return (r & 1) ? (r + 1) * G - 1 - c : r * G + c; }

__global__ void __launch_bounds__(kPPThreads, 1)
    attn_fwd_pp_kernel(const __grid_constant__ CUtensorMap tm_qkv, const AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023)) __trap();
  uint8_t* sQ = smem;                        // [2 tiles] x 32 KB
  uint8_t* sRing = sQ + 2 * TILE;            // kPPRing x 32 KB: K V K V ...
  float* sMax = (float*)(sRing + kPPRing * TILE);  // [2 tiles][2 parity][2 halves][128]
  uint64_t* bar = (uint64_t*)(sMax + 8 * AT);
  uint64_t* q_full = bar + 0;                // [2]
  uint64_t* q_empty = q_full + 2;            // [2] the tile's last S MMA of the item read Q
  uint64_t* t_full = q_empty + 2;            // [kPPRing]
  uint64_t* t_empty = t_full + kPPRing;      // [kPPRing]
  uint64_t* s_full = t_empty + kPPRing;      // [2] S_t(j) in TMEM
  uint64_t* p_full = s_full + 2;             // [2] P_t(j) written (8 warps)
  uint64_t* o_full = p_full + 2;             // [2] the tile's last P V of the item done
  uint32_t* tmem_slot = (uint32_t*)(o_full + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nqb = a.T / AT, npair = nqb / 2, Z = a.b * a.H, n_items = npair * Z;
  const int G = (int)gridDim.x, cta = (int)blockIdx.x;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    for (int t = 0; t < 2; ++t) {
      mbar_init(&q_full[t], 1);
      mbar_init(&q_empty[t], 1);
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 8);
      mbar_init(&o_full[t], 1);
    }
    for (int i = 0; i < kPPRing; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int slot = 0, ph = 0;
      for (int r = 0, it = 0;; ++r, ++it) {
        const int item = pp_item(r, cta, G);
        if (item >= n_items) break;
        const int p = npair - 1 - item / Z, z = item % Z;
        const int s = z / a.H, h = z % a.H, row0 = s * a.T;
        const int kcol = a.d + h * AT, vcol = 2 * a.d + h * AT;
        for (int t = 0; t < 2; ++t) {
          mbar_wait(&q_empty[t], (it & 1) ^ 1);
          mbar_arrive_expect_tx(&q_full[t], TILE);
          for (int c = 0; c < 2; ++c)
            tma_load_2d(sQ + t * TILE + c * CHUNK, &tm_qkv, &q_full[t], h * AT + 64 * c, row0 + (2 * p + t) * AT);
        }
        for (int n = 0; n < 2 * (2 * p + 2); ++n) {  // K_j (n = 2j), V_j (n = 2j+1), j = 0 .. 2p+1
          mbar_wait(&t_empty[slot], ph ^ 1);
          mbar_arrive_expect_tx(&t_full[slot], TILE);
          const int col = (n & 1) ? vcol : kcol;
          for (int c = 0; c < 2; ++c)
            tma_load_2d(sRing + slot * TILE + c * CHUNK, &tm_qkv, &t_full[slot], col + 64 * c, row0 + (n >> 1) * AT);
          if (++slot == kPPRing) {
            slot = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ring tile n (global, counted over items) sits in slot n % kPPRing with
    // phase (n / kPPRing) & 1; item tile counter n0 advances by 2 (2p + 2)
    int n0 = 0, gA = 0, gB = 0;  // ring tiles and per-tile blocks of the items before this one
    for (int r = 0, it = 0;; ++r, ++it) {
      const int item = pp_item(r, cta, G);
      if (item >= n_items) break;
      const int p = npair - 1 - item / Z;
      const int nb = 2 * p + 2;  // key blocks of tile B (tile A: nb - 1)
      auto kslot = [&](int j) { return (n0 + 2 * j) % kPPRing; };
      auto vslot = [&](int j) { return (n0 + 2 * j + 1) % kPPRing; };
      auto kph = [&](int j) { return (uint32_t)(((n0 + 2 * j) / kPPRing) & 1); };
      auto vph = [&](int j) { return (uint32_t)(((n0 + 2 * j + 1) / kPPRing) & 1); };
      auto issue_s = [&](int t, int j, bool release_k) {
        if (lane == 0) {
          const uint32_t aQ = smem_u32(sQ + t * TILE), aK = smem_u32(sRing + kslot(j) * TILE);
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            tc_mma_f16(tmem + t * 128, desc_kmajor(aQ, ks), desc_kmajor(aK, ks), idesc(0, 0), ks > 0 ? 1u : 0u);
          tc_commit(&s_full[t]);
          if (release_k) tc_commit(&t_empty[kslot(j)]);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int t, int j, bool release_v) {
        if (lane == 0) {
          const uint32_t aV = smem_u32(sRing + vslot(j) * TILE);
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            tc_mma_f16_ts(tmem + 256 + t * 128, tmem + t * 128 + 16 * ks, desc_mnmajor(aV, ks), idesc(0, 1),
                          (j > 0 || ks > 0) ? 1u : 0u);
          if (release_v) tc_commit(&t_empty[vslot(j)]);
        }
        __syncwarp();
      };
      mbar_wait(&q_full[0], it & 1);
      mbar_wait(&q_full[1], it & 1);
      mbar_wait(&t_full[kslot(0)], kph(0));
      tc_fence_after();
      issue_s(0, 0, false);
      issue_s(1, 0, true);
      for (int j = 0; j < nb; ++j) {
        const bool has_a = j < nb - 1;
        const bool last_a = j == nb - 2, last_b = j == nb - 1;
        mbar_wait(&t_full[vslot(j)], vph(j));
        if (has_a) {
          mbar_wait(&p_full[0], (gA + j) & 1);
          tc_fence_after();
          issue_pv(0, j, false);
          if (last_a) {
            if (lane == 0) {
              tc_commit(&o_full[0]);
              tc_commit(&q_empty[0]);
            }
            __syncwarp();
          } else {
            mbar_wait(&t_full[kslot(j + 1)], kph(j + 1));
            tc_fence_after();
            issue_s(0, j + 1, false);
          }
        }
        mbar_wait(&p_full[1], (gB + j) & 1);
        tc_fence_after();
        issue_pv(1, j, true);
        if (last_b) {
          if (lane == 0) {
            tc_commit(&o_full[1]);
            tc_commit(&q_empty[1]);
          }
          __syncwarp();
        } else {
          if (!has_a || last_a) {  // tile A done: K_{j+1} is B's alone
            mbar_wait(&t_full[kslot(j + 1)], kph(j + 1));
            tc_fence_after();
          }
          issue_s(1, j + 1, true);
        }
      }
      n0 += 2 * nb;
      gA += nb - 1;
      gB += nb;
    }
  } else {
    const int sw = warp - 2;                  // 0..15
    const int t = sw >> 3;                    // tile
    const int quad = warp & 3, half = (sw >> 2) & 1;
    const int r = quad * 32 + lane;
    const uint32_t lanes = (uint32_t)(quad * 32) << 16;
    const uint32_t tS = tmem + t * 128 + lanes, tO = tmem + 256 + t * 128 + lanes;
    const float c2 = a.scale * kLog2e;
    const int row_bar = 1 + t * 4 + quad;
    float* mxb = sMax + t * 4 * AT;           // this tile's [2 parity][2 halves][128]
    int g = 0;                                // this tile's blocks so far (barrier phases, sMax parity)
    for (int rr = 0, it = 0;; ++rr, ++it) {
      const int item = pp_item(rr, cta, G);
      if (item >= n_items) break;
      const int p = npair - 1 - item / Z, z = item % Z;
      const int s = z / a.H, h = z % a.H, row0 = s * a.T;
      const int qb = 2 * p + t;               // this tile's query block
      const int qi = qb * AT + r;
      float mref = -INFINITY, l = 0.f;
      for (int j = 0; j <= qb; ++j, ++g) {
        mbar_wait(&s_full[t], g & 1);
        tc_fence_after();
        // pass 1: the row max of this half (32 columns at a time, registers
        // reused; TMEM is read again in pass 2 instead of holding 64 values)
        const int lim = (j == qb) ? qi - (j * AT + half * 64) : 1 << 20;  // last visible column
        float cm = -INFINITY;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t rv[32];
          tmem_ld32(tS + half * 64 + 32 * c, rv);
          tmem_ld_wait_regs(rv);
#pragma unroll
          for (int u = 0; u < 32; ++u)
            if (32 * c + u <= lim) cm = fmaxf(cm, __uint_as_float(rv[u]));
        }
        float* mx = mxb + (g & 1) * 2 * AT;
        mx[half * AT + r] = cm;
        named_sync(row_bar, 64);
        const float mb = fmaxf(mx[r], mx[AT + r]) * c2;
        const bool resc = mb > mref + 8.f;
        float alpha = 1.f;
        if (resc) {
          alpha = ex2(mref - mb);
          mref = mb;
        }
        // O_t is stable here: S_t(j) was issued after P_t(j-1) V_{j-1}
        if (j > 0 && __any_sync(0xffffffffu, resc)) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint32_t o[32];
            tmem_ld32(tO + half * 64 + 32 * c, o);
            tmem_ld_wait_regs(o);
#pragma unroll
            for (int u = 0; u < 32; ++u) o[u] = __float_as_uint(__uint_as_float(o[u]) * alpha);
            tmem_st32(tO + half * 64 + 32 * c, o);
          }
        }
        // pass 2: P = 2^(S c2 - mref) -> bf16 pairs over the S columns just read
        float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t rv[32];
          tmem_ld32(tS + half * 64 + 32 * c, rv);
          tmem_ld_wait_regs(rv);
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {      // 16 keys = one k-step of P V
            uint32_t pk[8];
#pragma unroll
            for (int u = 0; u < 16; u += 2) {
              const int col = 32 * c + 16 * kk + u;
              const float e0 = col <= lim ? ex2(fmaf(__uint_as_float(rv[16 * kk + u]), c2, -mref)) : 0.f;
              const float e1 = col + 1 <= lim ? ex2(fmaf(__uint_as_float(rv[16 * kk + u + 1]), c2, -mref)) : 0.f;
              if (u & 2) acc1 += e0 + e1; else acc0 += e0 + e1;
              pk[u >> 1] = pack_bf16x2(e0, e1);
            }
            tmem_st8(tS + 16 * (4 * half + 2 * c + kk), pk);
          }
        }
        l = l * alpha + (acc0 + acc1);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t]);
      }
      // epilogue: O / l -> bf16 (this half of the head dims), LSE (log2 units);
      // row sums through the parity buffer the last block did not use
      float* sL = mxb + (g & 1) * 2 * AT;
      sL[half * AT + r] = l;
      named_sync(row_bar, 64);
      const float ltot = sL[r] + sL[AT + r];
      named_sync(row_bar, 64);
      const float inv = 1.f / ltot;
      mbar_wait(&o_full[t], it & 1);
      tc_fence_after();
      bf16* orow = a.o + (size_t)(row0 + qi) * a.d + h * AT + half * 64;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t rv[32];
        tmem_ld32(tO + half * 64 + 32 * c, rv);
        tmem_ld_wait_regs(rv);
#pragma unroll
        for (int u = 0; u < 32; u += 8) {
          float v[8];
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) v[kk] = __uint_as_float(rv[u + kk]) * inv;
          st_bf16x8(orow + 32 * c + u, v);
        }
      }
      tc_fence_before();
      if (half == 0) a.lse[(size_t)z * a.T + qi] = mref + __log2f(ltot);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ============================================================== backward
// One CTA per (z, 128-key block kb), over 64-query blocks i >= 2 kb.
// TMEM columns: dK [0,128), dV [128,256), SP[2] [256,384) (S^T of block i,
// then P^T in bf16 pairs written over the columns each thread has read:
// k-step ks of dV += P^T dO_i reads columns [16 ks, 16 ks + 8)), DQ[2]
// [384,512) (dP^T of block i, then dQ_i^T = K^T dS_i^T once dP^T is read).
// With both double-buffered, the MMA warp issues S^T / dP^T of block i+1
// before it waits for the gradient warps to finish block i; four drain warps
// reduce-add dQ^T into an fp32 accumulator [z][head dim][T] (dq_finalize
// transposes it into dqkv) off the gradient warps' path.  Every MMA is
// M = 128.  Q_i / dO_i stream through 3 stages, dS^T is double-buffered.
constexpr int QB = 64;                 // queries per backward step
constexpr int QCHUNK = QB * 128;       // [64 rows x 64 cols] bf16 SWIZZLE_128B chunk (8 KB)
constexpr int QTILE = 2 * QCHUNK;      // [64 x 128] bf16
constexpr int NQS = 3;                 // Q_i / dO_i stages

__device__ __forceinline__ uint64_t desc_kmajor_c(uint32_t base, int ks, int chunk) {
  return umma_desc_sw128(base + (ks >> 2) * chunk + (ks & 3) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t desc_mnmajor_c(uint32_t base, int ks, int chunk) {
  return umma_desc_sw128(base + ks * 2048, chunk, 1024);
}
constexpr uint32_t idesc_n(int a_mn, int b_mn, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(AT >> 4) << 24);
}

// warp 0 TMA, warp 1 MMA, warps 2..17 gradient (4 per TMEM lane quadrant,
// 16 query columns each), warps 18..21 dQ^T drain (one per quadrant)
constexpr int kBwdThreads = 704;
constexpr int kBwdCols = QB / 4;

__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                    const __grid_constant__ CUtensorMap tm_do, const __grid_constant__ CUtensorMap tm_dq,
                    const AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;  // no static shared memory: the window starts 1024-aligned (checked)
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023)) __trap();
  uint8_t* sK = smem;                  // 32 KB
  uint8_t* sV = sK + TILE;             // 32 KB
  uint8_t* sQ = sV + TILE;             // NQS stages x 16 KB  (query block i)
  uint8_t* sdO = sQ + NQS * QTILE;     // NQS stages x 16 KB
  uint8_t* sdST = sdO + NQS * QTILE;   // 2 buffers x 16 KB  dS^T [128 keys x 64 queries]
  uint8_t* sStg = sdST + 2 * QTILE;    // 4 drain warps x 4 KB dQ^T staging
  float* sLse = (float*)(sStg + 4 * 4096);  // [NQS][64] (log2 units)
  float* sD = sLse + NQS * QB;              // [NQS][64]
  uint64_t* bar = (uint64_t*)(sD + NQS * QB);
  uint64_t* kv_full = bar + 0;
  uint64_t* qd_full = bar + 1;    // [NQS] Q_i, dO_i, LSE_i, D_i landed
  uint64_t* qd_empty = bar + 1 + NQS;   // [NQS] dV, dK of block i done
  uint64_t* s_full = bar + 1 + 2 * NQS;  // [2] S^T in SP[b]
  uint64_t* dp_full = s_full + 2;        // [2] dP^T in DQ[b]
  uint64_t* pd_full = dp_full + 2;       // [2] P^T (SP[b]), dS^T (smem) written; S^T, dP^T read (16 warps)
  uint64_t* pd_empty = pd_full + 2;      // [2] dK, dQ^T done reading dS^T (smem buffer b)
  uint64_t* dq_full = pd_empty + 2;      // [2] dQ^T in DQ[b]
  uint64_t* dq_empty = dq_full + 2;      // [2] dQ^T read (4 drain warps)
  uint64_t* kv_done = dq_empty + 2;      // dK, dV final
  uint32_t* tmem_slot = (uint32_t*)(kv_done + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nb = a.T / AT, Z = a.b * a.H;
  const long long cta_t0 = (a.diag & 0x400) ? gtimer() : 0;
  const int kb = (int)(blockIdx.x / Z);  // heavy (early) key blocks first
  const int z = blockIdx.x % Z;
  const int s = z / a.H, h = z % a.H;
  const int row0 = s * a.T;
  const int qcol = h * AT, kcol = a.d + h * AT, vcol = 2 * a.d + h * AT;
  const int i0 = 2 * kb, n_it = 2 * (nb - kb);  // 64-query blocks i0 .. i0 + n_it - 1
  const bool tr = (a.diag & 0x200) && blockIdx.x == 0 && lane == 0;
#define TRACE(it, ev) \
  if (tr && (it) < 64) a.trace[(it) * 16 + (ev)] = clock64();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_kv);
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_dq);
    mbar_init(kv_full, 1);
    for (int k = 0; k < NQS; ++k) {
      mbar_init(&qd_full[k], 1);
      mbar_init(&qd_empty[k], 1);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&s_full[k], 1);
      mbar_init(&dp_full[k], 1);
      mbar_init(&pd_full[k], 16);
      mbar_init(&dq_full[k], 1);
      mbar_init(&dq_empty[k], 4);
      mbar_init(&pd_empty[k], 1);
    }
    mbar_init(kv_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tdK = tmem, tdV = tmem + 128, tSP = tmem + 256, tDQ = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * TILE);
      for (int c = 0; c < 2; ++c) {
        tma_load_2d(sK + c * CHUNK, &tm_kv, kv_full, kcol + 64 * c, row0 + kb * AT);
        tma_load_2d(sV + c * CHUNK, &tm_kv, kv_full, vcol + 64 * c, row0 + kb * AT);
      }
      for (int it = 0, st = 0, ph = 0; it < n_it; ++it) {
        const int i = i0 + it;
        mbar_wait(&qd_empty[st], ph ^ 1);
        TRACE(it, 0)
        if (a.diag & 8) {
          mbar_arrive(&qd_full[st]);
          if (++st == NQS) {
            st = 0;
            ph ^= 1;
          }
          continue;
        }
        mbar_arrive_expect_tx(&qd_full[st], 2 * QTILE + 2 * QB * 4);
        for (int c = 0; c < 2; ++c) {
          tma_load_2d(sQ + st * QTILE + c * QCHUNK, &tm_q, &qd_full[st], qcol + 64 * c, row0 + i * QB);
          tma_load_2d(sdO + st * QTILE + c * QCHUNK, &tm_do, &qd_full[st], h * AT + 64 * c, row0 + i * QB);
        }
        bulk_g2s(sLse + st * QB, a.lse + (size_t)z * a.T + i * QB, QB * 4, &qd_full[st]);
        bulk_g2s(sD + st * QB, a.D + (size_t)z * a.T + i * QB, QB * 4, &qd_full[st]);
        if (++st == NQS) {
          st = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    mbar_wait(kv_full, 0);
    tc_fence_after();
    const uint32_t aK = smem_u32(sK), aV = smem_u32(sV);
    // S^T = K Q_i^T -> SP[b], dP^T = V dO_i^T -> DQ[b] (stage st landed)
    auto issue_sdp = [&](int b, int st, bool do_dp) {
      if (lane == 0) {
        const uint32_t aQ = smem_u32(sQ + st * QTILE), adO = smem_u32(sdO + st * QTILE);
        if (!(a.diag & 0x14)) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            tc_mma_f16(tSP + b * QB, desc_kmajor(aK, ks), desc_kmajor_c(aQ, ks, QCHUNK), idesc_n(0, 0, QB),
                       ks > 0 ? 1u : 0u);
        }
        tc_commit(&s_full[b]);
        if (do_dp) {
          if (!(a.diag & 0x24)) {
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
              tc_mma_f16(tDQ + b * QB, desc_kmajor(aV, ks), desc_kmajor_c(adO, ks, QCHUNK), idesc_n(0, 0, QB),
                         ks > 0 ? 1u : 0u);
          }
          tc_commit(&dp_full[b]);
        }
      }
      __syncwarp();
    };
    auto issue_dp = [&](int b, int st) {
      if (lane == 0) {
        const uint32_t adO = smem_u32(sdO + st * QTILE);
        if (!(a.diag & 0x24)) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            tc_mma_f16(tDQ + b * QB, desc_kmajor(aV, ks), desc_kmajor_c(adO, ks, QCHUNK), idesc_n(0, 0, QB),
                       ks > 0 ? 1u : 0u);
        }
        tc_commit(&dp_full[b]);
      }
      __syncwarp();
    };
    mbar_wait(&qd_full[0], 0);
    tc_fence_after();
    issue_sdp(0, 0, true);
    for (int it = 0, st = 0, ph = 0; it < n_it; ++it) {
      const int nst = st + 1 == NQS ? 0 : st + 1, nph = st + 1 == NQS ? ph ^ 1 : ph;
      const int b = it & 1, nbuf = b ^ 1;
      if (it + 1 < n_it) {
        // SP[nbuf]: S^T(it-1) read and P^T(it-1) consumed by dV(it-1), issued earlier (in-order pipe)
        mbar_wait(&qd_full[nst], nph);
        TRACE(it, 1)
        tc_fence_after();
        issue_sdp(nbuf, nst, false);
        // DQ[nbuf]: dP^T(it-1) read (pd_full(it-1) seen) and dQ^T(it-1) drained
        if (it >= 1) mbar_wait(&dq_empty[nbuf], ((it - 1) >> 1) & 1);
        TRACE(it, 2)
        tc_fence_after();
        issue_dp(nbuf, nst);
      }
      mbar_wait(&pd_full[b], (it >> 1) & 1);  // P^T, dS^T of block it written; S^T, dP^T read
      TRACE(it, 3)
      tc_fence_after();
      if (lane == 0) {
        const uint32_t acc = it > 0 ? 1u : 0u;
        const uint32_t aQ = smem_u32(sQ + st * QTILE), adO = smem_u32(sdO + st * QTILE);
        const uint32_t adST = smem_u32(sdST + b * QTILE);
#pragma unroll
        for (int ks = 0; ks < QB / 16; ++ks) {
          // dV += P^T dO_i (A from TMEM) ; dK += dS^T Q_i  (K = 64 queries; B read MN-major)
          if (!(a.diag & 0x44))
            tc_mma_f16_ts(tdV, tSP + b * QB + 16 * ks, desc_mnmajor_c(adO, ks, QCHUNK), idesc_n(0, 1, AT),
                          (acc || ks > 0) ? 1u : 0u);
          if (!(a.diag & 0x84))
            tc_mma_f16(tdK, desc_kmajor(adST, ks), desc_mnmajor_c(aQ, ks, QCHUNK), idesc_n(0, 1, AT),
                       (acc || ks > 0) ? 1u : 0u);
        }
        tc_commit(&qd_empty[st]);
        if (!(a.diag & 0x104)) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)  // dQ_i^T = K^T dS_i^T  (both operands MN-major, K = 128 keys)
            tc_mma_f16(tDQ + b * QB, desc_mnmajor(aK, ks), desc_mnmajor_c(adST, ks, QCHUNK), idesc_n(1, 1, QB),
                       ks > 0 ? 1u : 0u);
        }
        tc_commit(&dq_full[b]);
        tc_commit(&pd_empty[b]);
      }
      __syncwarp();
      st = nst;
      ph = nph;
    }
    if (lane == 0) tc_commit(kv_done);
    __syncwarp();
  } else if (warp < 18) {
    // gradient warps: lane quadrant quad, query-column group cg (16 of the 64)
    const int quad = warp & 3, cg = (warp - 2) >> 2;
    const int r = quad * 32 + lane;  // key row (S^T, dP^T, P^T, dK, dV)
    const int kj = kb * AT + r;      // key position
    const uint32_t lanes = (uint32_t)(quad * 32) << 16;
    const float c2 = a.scale * kLog2e;
    for (int it = 0, st = 0, ph = 0; it < n_it; ++it) {
      const int i = i0 + it, b = it & 1;
      const uint32_t bph = (it >> 1) & 1;
      const uint32_t tS = tSP + b * QB + lanes + cg * kBwdCols;
      mbar_wait(&s_full[b], bph);
      if (warp == 2) TRACE(it, 4)
      tc_fence_after();
      uint32_t rs[16];
      tmem_ld16(tS, rs);
      tmem_ld_wait_regs16(rs);
      if (a.diag & 2) {
        mbar_wait(&dp_full[b], bph);
        if (warp == 2) TRACE(it, 5)
        mbar_wait(&pd_empty[b], bph ^ 1);
        if (warp == 2) TRACE(it, 6)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pd_full[b]);
        if (++st == NQS) {
          st = 0;
          ph ^= 1;
        }
        continue;
      }
      mbar_wait(&qd_full[st], ph);  // LSE_i, D_i landed (the MMA warp saw it before S^T)
      const float* lse = sLse + st * QB + cg * kBwdCols;
      const float* Dq = sD + st * QB + cg * kBwdCols;
      float p[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) p[t] = ex2(fmaf(__uint_as_float(rs[t]), c2, -lse[t]));
      if (it < 2) {  // diagonal: queries before this key are masked
        const int lim = kj - (i * QB + cg * kBwdCols);
#pragma unroll
        for (int t = 0; t < 16; ++t)
          if (t < lim) p[t] = 0.f;
      }
      if (warp == 2) TRACE(it, 10)
      mbar_wait(&dp_full[b], bph);
      if (warp == 2) TRACE(it, 5)
      tc_fence_after();
      tmem_ld16(tDQ + b * QB + lanes + cg * kBwdCols, rs);
      tmem_ld_wait_regs16(rs);
      uint32_t pkp[8], pkd[8];  // P^T, dS^T row pieces as bf16x2
#pragma unroll
      for (int t = 0; t < 16; t += 2) {
        const float d0 = p[t] * (__uint_as_float(rs[t]) - Dq[t]);
        const float d1 = p[t + 1] * (__uint_as_float(rs[t + 1]) - Dq[t + 1]);
        pkp[t >> 1] = pack_bf16x2(p[t], p[t + 1]);
        pkd[t >> 1] = pack_bf16x2(d0, d1);
      }
      // P^T over this thread's own S^T columns (k-step cg of dV); dS^T to smem
      tmem_st8(tS, pkp);
      if (warp == 2) TRACE(it, 11)
      mbar_wait(&pd_empty[b], bph ^ 1);  // dK, dQ^T of block it-2 done with dS^T buffer b
      if (warp == 2) TRACE(it, 6)
      {
        const uint32_t row = smem_u32(sdST + b * QTILE) + r * 128;
        const int p0 = cg * 2;  // first 16-byte piece (8 queries) of this column group
        sts128(row + ((p0 ^ (r & 7)) << 4), pkd[0], pkd[1], pkd[2], pkd[3]);
        sts128(row + (((p0 + 1) ^ (r & 7)) << 4), pkd[4], pkd[5], pkd[6], pkd[7]);
      }
      tmem_st_wait();
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (warp == 2) TRACE(it, 7)
      if (lane == 0) mbar_arrive(&pd_full[b]);
      if (++st == NQS) {
        st = 0;
        ph ^= 1;
      }
    }
    // dK (scaled), dV -> bf16 into dqkv (k and v sections), thread = key row, 32 columns
    mbar_wait(kv_done, 0);
    tc_fence_after();
    for (int which = 0; which < 2; ++which) {
      const uint32_t tb = (which == 0 ? tdK : tdV) + lanes + cg * 32;
      bf16* out = a.dqkv + (size_t)(row0 + kj) * 3 * a.d + (which == 0 ? a.d : 2 * a.d) + h * AT + cg * 32;
      const float sc = which == 0 ? a.scale : 1.f;
      uint32_t r0[32];
      tmem_ld32(tb, r0);
      tmem_ld_wait_regs(r0);
      float v[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) v[t] = __uint_as_float(r0[t]) * sc;
#pragma unroll
      for (int t = 0; t < 32; t += 8) st_bf16x8(out + t, v + t);
    }
  } else {
    // drain warps: dQ^T rows of lane quadrant quad (head dims), 64 queries in 2 chunks of 32
    const int quad = warp & 3;
    const uint32_t lanes = (uint32_t)(quad * 32) << 16;
    uint8_t* stg = sStg + (warp - 18) * 4096;
    for (int it = 0; it < n_it; ++it) {
      const int b = it & 1;
      mbar_wait(&dq_full[b], (it >> 1) & 1);
      if (warp == 18) TRACE(it, 8)
      tc_fence_after();
      uint32_t r0[32], r1[32];
      tmem_ld32(tDQ + b * QB + lanes, r0);
      tmem_ld32(tDQ + b * QB + lanes + 32, r1);
      tmem_ld_wait_regs(r0);
      tmem_ld_wait_regs(r1);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dq_empty[b]);
      if (warp == 18) TRACE(it, 9)
      auto stage = [&](const uint32_t(&rq)[32], int c) {
        if (lane == 0) bulk_wait_read<0>();  // the previous reduce has read the staging buffer
        __syncwarp();
        const uint32_t frow = smem_u32(stg) + lane * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          sts128(frow + ((q ^ (lane & 7)) << 4), __float_as_uint(__uint_as_float(rq[4 * q]) * a.scale),
                 __float_as_uint(__uint_as_float(rq[4 * q + 1]) * a.scale),
                 __float_as_uint(__uint_as_float(rq[4 * q + 2]) * a.scale),
                 __float_as_uint(__uint_as_float(rq[4 * q + 3]) * a.scale));
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (!(a.diag & 3)) tma_reduce_add_2d(&tm_dq, stg, (i0 + it) * QB + c * 32, z * AT + quad * 32);
          bulk_commit();
        }
      };
      stage(r0, 0);
      stage(r1, 1);
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
  if ((a.diag & 0x400) && threadIdx.x == 0) {
    a.cta[3 * blockIdx.x] = smid();
    a.cta[3 * blockIdx.x + 1] = cta_t0;
    a.cta[3 * blockIdx.x + 2] = gtimer();
  }
#undef TRACE
}

// dQ^T (fp32 accumulator [z][head dim][T]) -> bf16 q section of dqkv
// ([b*T, 3d], row s*T + t, column h*128 + c); clears the accumulator.  One
// block per (z, 64 positions): all 16 loads per thread are issued before any
// store (coalesced 256 B row pieces along t), then 16 B writes along c.
constexpr int kFinT = 64;
__global__ void __launch_bounds__(256) dq_finalize_kernel(float* __restrict__ acc, bf16* __restrict__ dqkv, int H,
                                                          int T, int d) {
  __shared__ float tile[AT][kFinT + 1];
  const int z = blockIdx.y, t0 = blockIdx.x * kFinT;
  const int s = z / H, h = z % H;
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  float2* src = reinterpret_cast<float2*>(acc + (size_t)z * AT * T + t0) + lane;
  const int T2 = T / 2;
  float2 v[AT / 8];
#pragma unroll
  for (int k = 0; k < AT / 8; ++k) v[k] = src[(size_t)(w + 8 * k) * T2];
#pragma unroll
  for (int k = 0; k < AT / 8; ++k) {
    tile[w + 8 * k][2 * lane] = v[k].x;
    tile[w + 8 * k][2 * lane + 1] = v[k].y;
  }
#pragma unroll
  for (int k = 0; k < AT / 8; ++k) src[(size_t)(w + 8 * k) * T2] = make_float2(0.f, 0.f);
  __syncthreads();
#pragma unroll
  for (int k = threadIdx.x; k < kFinT * (AT / 8); k += 256) {
    const int t = k / (AT / 8), c0 = (k % (AT / 8)) * 8;
    uint4 u;
    u.x = pack_bf16x2(tile[c0 + 0][t], tile[c0 + 1][t]);
    u.y = pack_bf16x2(tile[c0 + 2][t], tile[c0 + 3][t]);
    u.z = pack_bf16x2(tile[c0 + 4][t], tile[c0 + 5][t]);
    u.w = pack_bf16x2(tile[c0 + 6][t], tile[c0 + 7][t]);
    *reinterpret_cast<uint4*>(dqkv + (size_t)(s * T + t0 + t) * 3 * d + h * AT + c0) = u;
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

static_assert(FwdCfg<2>::kSmem <= 232448 && FwdCfg<4>::kSmem <= 232448, "attn fwd shared memory");
constexpr int kBwdSmem = 2 * TILE + (2 * NQS + 2) * QTILE + 4 * 4096 + 2 * NQS * QB * 4 + 256;
static_assert(kBwdSmem <= 232448, "attn bwd shared memory");

// diag 0x400: per-CTA occupancy summary of one launch (third call of each kernel)
static void cta_summary(const char* name, long long* dev, int n, int blocks_of(int), cudaStream_t st) {
  static int calls[2] = {0, 0};
  const int k = name[5] == 'f' ? 0 : 1;
  if (calls[k]++ != 2) return;
  std::vector<long long> h(3 * (size_t)n);
  cudaStreamSynchronize(st);
  cudaMemcpy(h.data(), dev, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
  long long t0 = h[1], t1 = h[2], busy = 0;
  for (int i = 0; i < n; ++i) {
    t0 = std::min(t0, h[3 * i + 1]);
    t1 = std::max(t1, h[3 * i + 2]);
    busy += h[3 * i + 2] - h[3 * i + 1];
  }
  fprintf(stderr, "%s ctas %d span %.2f us  sum cta %.2f us  occupancy(148 SM) %.3f\n", name, n, (t1 - t0) / 1e3,
          busy / 1e3, busy / (148.0 * (t1 - t0)));
  // per work size: mean duration, mean start
  std::vector<double> dsum(64, 0), ssum(64, 0), esum(64, 0);
  std::vector<int> cnt(64, 0);
  for (int i = 0; i < n; ++i) {
    int w = blocks_of(i);
    if (w < 0 || w >= 64) continue;
    dsum[w] += h[3 * i + 2] - h[3 * i + 1];
    ssum[w] += h[3 * i + 1] - t0;
    esum[w] += h[3 * i + 2] - t0;
    cnt[w]++;
  }
  for (int w = 0; w < 64; ++w)
    if (cnt[w])
      fprintf(stderr, "  blocks %2d: n %3d  dur %7.2f us  start %7.2f  end %7.2f\n", w, cnt[w], dsum[w] / cnt[w] / 1e3,
              ssum[w] / cnt[w] / 1e3, esum[w] / cnt[w] / 1e3);
}
static int g_nqb = 16, g_Z = 16, g_G = 148;
static int fwd_blocks(int c) {  // total key blocks of persistent CTA c (snake deal, as fwd_item)
  int tot = 0;
  for (int r = 0;; ++r) {
    const int i = (r & 1) ? (r + 1) * g_G - 1 - c : r * g_G + c;
    if (i >= g_nqb * g_Z) break;
    tot += g_nqb - i / g_Z;
  }
  return tot;
}
static int bwd_blocks(int i) { return g_nqb - (i / g_Z); }

// SMs the persistent attention forward may use (adaptra_set_tuning
// ADAPTRA_TUNE_ATTN_SMS; 0 = all)
std::atomic<int> g_attn_sms{0};

int attn_fwd_tc(const bf16* qkv, bf16* o, float* lse, int b, int H, int T, int d, cudaStream_t st) {
  if (d != H * AT || T % AT) return set_error(ADAPTRA_EINVAL, "attn_fwd_tc: head dim 128 and T % 128 required");
  CUtensorMap m;
  int rc = map2d(&m, qkv, (int64_t)b * T, 3LL * d, 3LL * d, 2, 64, AT, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  static const int nq = [] {
    const char* v = getenv("ADAPTRA_ATTN_FWD_WARPS");
    return (v && atoi(v) == 16) ? 4 : 2;
  }();
  // exponentials per 4 on the FMA pipe (ex2_poly): $ADAPTRA_ATTN_POLY = 0 | 1 | 2
  static const int poly = [] {
    const char* v = getenv("ADAPTRA_ATTN_POLY");
    return v ? std::max(0, std::min(2, atoi(v))) : 0;
  }();
  static std::atomic<unsigned> attr{0};  // per device; stage threads may race here
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr.load(std::memory_order_acquire) & (1u << dev))) {
    cudaFuncSetAttribute(attn_fwd_kernel<2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdCfg<2>::kSmem);
    cudaFuncSetAttribute(attn_fwd_kernel<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdCfg<2>::kSmem);
    cudaFuncSetAttribute(attn_fwd_kernel<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdCfg<2>::kSmem);
    cudaFuncSetAttribute(attn_fwd_kernel<4, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdCfg<4>::kSmem);
    cudaFuncSetAttribute(attn_fwd_kernel<2, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdCfg<2>::kSmem);
    cudaFuncSetAttribute(attn_fwd_kernel<2, 0, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdCfg<2>::kSmem);
    cudaFuncSetAttribute(attn_fwd_kernel<2, 0, 2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdCfg<2>::kSmem);
    cudaFuncSetAttribute(attn_fwd_kernel<2, 0, 1, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdCfg<2>::kSmem);
    cudaFuncSetAttribute(attn_fwd_kernel<4, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdCfg<4>::kSmem);
    cudaFuncSetAttribute(attn_fwd_kernel<2, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdCfg<2>::kSmem);
    cudaFuncSetAttribute(attn_fwd_kernel<2, 2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdCfg<2>::kSmem);
    cudaFuncSetAttribute(attn_fwd_pp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPPSmem);
    attr.fetch_or(1u << dev, std::memory_order_release);
  }
  AttnArgs a{};
  a.b = b; a.H = H; a.T = T; a.d = d;
  a.scale = 1.f / std::sqrt((float)AT);
  a.o = o;
  a.lse = lse;
  void* pb = prof_on() ? prof_begin(st) : nullptr;
  static const int fdiag = getenv("ADAPTRA_ATTN_DIAG") ? atoi(getenv("ADAPTRA_ATTN_DIAG")) : 0;
  a.diag = fdiag & 0x600;
  static long long* ftrace = nullptr;
  if ((fdiag & 0x200) && !ftrace) cudaMalloc(&ftrace, 64 * 16 * sizeof(long long));
  a.trace = ftrace;
  static long long* fcta = nullptr;
  if ((fdiag & 0x400) && !fcta) cudaMalloc(&fcta, 3 * 4096 * sizeof(long long));
  a.cta = fcta;
  static int n_sm[32] = {0};
  if (!n_sm[dev & 31]) cudaDeviceGetAttribute(&n_sm[dev & 31], cudaDevAttrMultiProcessorCount, dev);
  // ADAPTRA_ATTN_FWD_GRID=items: one CTA per item (the non-persistent launch, for comparison)
  static const bool per_item = getenv("ADAPTRA_ATTN_FWD_GRID") && !strcmp(getenv("ADAPTRA_ATTN_FWD_GRID"), "items");
  const int sm_cap = g_attn_sms.load(std::memory_order_relaxed);
  const int n_use = (sm_cap > 0 && sm_cap < n_sm[dev & 31]) ? sm_cap : n_sm[dev & 31];
  const int items = b * H * (T / AT), grid = per_item ? items : std::min(items, n_use);
  // ping-pong over query-block pairs: opt-in ($ADAPTRA_ATTN_FWD=pp; needs an
  // even number of query blocks).  Correct (parity tests), but measured 1.75x
  // slower than the one-tile kernel on C1 shapes (56 vs 32 us per launch,
  // profiles/r02_op_bench_pp.jsonl): two softmax groups sharing the SM's
  // MUFU / issue slots plus the second TMEM pass cost more than the overlap gains
  static const bool pp_on = getenv("ADAPTRA_ATTN_FWD") && !strcmp(getenv("ADAPTRA_ATTN_FWD"), "pp");
  // P kept in TMEM for P V ($ADAPTRA_ATTN_FWD=ptmem; 30.2 vs 32.7 us per C1
  // launch, profiles/r02_attn_ptmem_ab.jsonl).  Opt-in, not the default: with
  // eight stages sharing the GPU the 8-stage bench hung in 3 of 6 runs on it
  // (0 of 4 with P through shared memory, profiles/r02_attn_ptmem_hang.txt);
  // its parity tests pass.  The variants built on it (qtmem, sep, s2) share
  // that status.
  static const bool p_tmem = getenv("ADAPTRA_ATTN_FWD") && !strcmp(getenv("ADAPTRA_ATTN_FWD"), "ptmem");
  // Q kept in TMEM as well ($ADAPTRA_ATTN_FWD=qtmem)
  static const bool q_tmem = getenv("ADAPTRA_ATTN_FWD") && !strcmp(getenv("ADAPTRA_ATTN_FWD"), "qtmem");
  // one S buffer released at load, P in separate buffers, Q in TMEM ($ADAPTRA_ATTN_FWD=sep)
  static const bool sep_p = getenv("ADAPTRA_ATTN_FWD") && !strcmp(getenv("ADAPTRA_ATTN_FWD"), "sep");
  // S and P V from two issuing warps ($ADAPTRA_ATTN_FWD=s2)
  static const bool s2 = getenv("ADAPTRA_ATTN_FWD") && !strcmp(getenv("ADAPTRA_ATTN_FWD"), "s2");
  if (pp_on && (T / AT) % 2 == 0 && !per_item) {
    const int pitems = b * H * (T / AT) / 2;
    attn_fwd_pp_kernel<<<std::min(pitems, n_use), kPPThreads, kPPSmem, st>>>(m, a);
  } else if (s2 && nq == 2 && poly == 0) {
    attn_fwd_kernel<2, 0, 1, 0, 1><<<grid, FwdCfg<2>::kThreads + 32, FwdCfg<2>::kSmem, st>>>(m, a);
  } else if (sep_p && nq == 2 && poly == 0) {
    attn_fwd_kernel<2, 0, 2, 1><<<grid, FwdCfg<2>::kThreads + 128, FwdCfg<2>::kSmem, st>>>(m, a);
  } else if (q_tmem && nq == 2 && poly == 0) {
    attn_fwd_kernel<2, 0, 1, 1><<<grid, FwdCfg<2>::kThreads + 128, FwdCfg<2>::kSmem, st>>>(m, a);
  } else if (p_tmem && nq == 2 && poly == 0) {
    attn_fwd_kernel<2, 0, 1><<<grid, FwdCfg<2>::kThreads, FwdCfg<2>::kSmem, st>>>(m, a);
  } else if (p_tmem && nq == 2 && poly == 1) {
    attn_fwd_kernel<2, 1, 1><<<grid, FwdCfg<2>::kThreads, FwdCfg<2>::kSmem, st>>>(m, a);
  } else if (p_tmem && nq == 2 && poly == 2) {
    attn_fwd_kernel<2, 2, 1><<<grid, FwdCfg<2>::kThreads, FwdCfg<2>::kSmem, st>>>(m, a);
  } else if (nq == 4 && p_tmem) {
    attn_fwd_kernel<4, 0, 1><<<grid, FwdCfg<4>::kThreads, FwdCfg<4>::kSmem, st>>>(m, a);
  } else if (nq == 4) {
    attn_fwd_kernel<4, 0><<<grid, FwdCfg<4>::kThreads, FwdCfg<4>::kSmem, st>>>(m, a);
  } else if (poly == 2) {
    attn_fwd_kernel<2, 2><<<grid, FwdCfg<2>::kThreads, FwdCfg<2>::kSmem, st>>>(m, a);
  } else if (poly == 1) {
    attn_fwd_kernel<2, 1><<<grid, FwdCfg<2>::kThreads, FwdCfg<2>::kSmem, st>>>(m, a);
  } else {
    attn_fwd_kernel<2, 0><<<grid, FwdCfg<2>::kThreads, FwdCfg<2>::kSmem, st>>>(m, a);
  }
  if (fdiag & 0x400) {
    g_nqb = T / AT; g_Z = b * H; g_G = grid;
    cta_summary("attn_fwd", fcta, grid, fwd_blocks, st);
  }
  if (fdiag & 0x200) {
    static int fdumped = 0;
    long long hb[64 * 16];
    cudaStreamSynchronize(st);
    cudaMemcpy(hb, ftrace, sizeof(hb), cudaMemcpyDeviceToHost);
    if (fdumped++ == 2) {
      for (int g = 0; g < 32; ++g) {
        fprintf(stderr, "fwd g %2d", g);
        for (int e = 0; e < 9; ++e) fprintf(stderr, " %7lld", hb[g * 16 + e] - hb[0]);
        fprintf(stderr, "\n");
      }
    }
  }
  if (pb) {
    double fl = 4.0 * (double)T * T * AT * b * H * 0.5;  // algorithmic: QK^T + PV, causal half (R28)
    prof_end(pb, st, PROF_ATTN, fl, 0);
  }
  return check_launch("attn_fwd_tc");
}

int attn_bwd_tc(const bf16* qkv, const bf16* dO, const float* lse, const float* D, bf16* dqkv, float* dq_acc, int b,
                int H, int T, int d, cudaStream_t st) {
  if (d != H * AT || T % AT) return set_error(ADAPTRA_EINVAL, "attn_bwd_tc: head dim 128 and T % 128 required");
  CUtensorMap mkv, mq, mdo, mdq;
  int rc = map2d(&mkv, qkv, (int64_t)b * T, 3LL * d, 3LL * d, 2, 64, AT, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = map2d(&mq, qkv, (int64_t)b * T, 3LL * d, 3LL * d, 2, 64, QB, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = map2d(&mdo, dO, (int64_t)b * T, d, d, 2, 64, QB, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = map2d(&mdq, dq_acc, (int64_t)b * H * AT, T, T, 4, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  static std::atomic<unsigned> attr{0};  // per device; stage threads may race here
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr.load(std::memory_order_acquire) & (1u << dev))) {
    cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdSmem);
    attr.fetch_or(1u << dev, std::memory_order_release);
  }
  AttnArgs a{};
  a.b = b; a.H = H; a.T = T; a.d = d;
  a.scale = 1.f / std::sqrt((float)AT);
  a.lse = const_cast<float*>(lse);
  a.D = D;
  a.dqkv = dqkv;
  a.dq_acc = dq_acc;
  void* pb = prof_on() ? prof_begin(st) : nullptr;
  static const int diag = getenv("ADAPTRA_ATTN_DIAG") ? atoi(getenv("ADAPTRA_ATTN_DIAG")) : 0;
  a.diag = diag;
  static long long* trace = nullptr;
  if ((diag & 0x200) && !trace) cudaMalloc(&trace, 64 * 16 * sizeof(long long));
  a.trace = trace;
  static long long* bcta = nullptr;
  if ((diag & 0x400) && !bcta) cudaMalloc(&bcta, 3 * 4096 * sizeof(long long));
  a.cta = bcta;
  attn_bwd_kernel<<<b * H * (T / AT), kBwdThreads, kBwdSmem, st>>>(mkv, mq, mdo, mdq, a);
  if (diag & 0x400) {
    g_nqb = T / AT; g_Z = b * H;
    cta_summary("attn_bwd", bcta, b * H * (T / AT), bwd_blocks, st);
  }
  if (diag & 0x200) {
    static int dumped = 0;
    long long h[64 * 16];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
    if (dumped++ == 2) {
      for (int it = 0; it < 32; ++it) {
        fprintf(stderr, "it %2d", it);
        for (int e = 0; e < 12; ++e) fprintf(stderr, " %7lld", h[it * 16 + e] - h[0]);
        fprintf(stderr, "\n");
      }
    }
  }
  if (pb) {
    double fl = 8.0 * (double)T * T * AT * b * H * 0.5;  // dP, dV, dK, dQ (causal half)
    prof_end(pb, st, PROF_ATTN_BWD, fl, 0);
  }
  rc = check_launch("attn_bwd_tc");
  if (rc) return rc;
  dq_finalize_kernel<<<dim3(T / kFinT, b * H), 256, 0, st>>>(dq_acc, dqkv, H, T, d);
  return check_launch("dq_finalize");
}

}  // namespace adaptra
