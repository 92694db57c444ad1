// tcgen05 / TMEM / TMA bf16 GEMM for sm_100a (stage F, B = dX and W = dW
// contractions, and the batched attention products).
//
// Persistent warp-specialised kernel, one CTA per SM (CG = 1) or one CTA pair
// per 2 SMs (CG = 2, tcgen05 cta_group::2: a 256 x BN tile whose A rows and B
// rows are split over the two CTAs' shared memory, MMA issued by the leader):
//   warps 0..7  epilogue (two warpgroups, setmaxnreg 208): tcgen05.ld TMEM ->
//               registers -> fused epilogue (bias / GeLU / residual / dGeLU /
//               row-dot; residual and GeLU inputs arrive by TMA) -> swizzled
//               shared-memory staging -> TMA store / TMA reduce-add
//   warp 8      TMA producer (one elected lane) -> smem ring of kStages stages
//   warp 9      TMEM allocator + MMA issuer (one elected lane, tcgen05.mma
//               kind::f16, (128 CG) x BN x 16 per instruction, fp32 accumulate)
//   warps 10,11 idle (complete the setmaxnreg-decreased warpgroup); in the
//               grouped dW kernel warp 10 sums the dY tiles into db
// Two TMEM accumulators (2 x BN columns) let the epilogue of tile t overlap
// the main loop of tile t+1.  gemm_tc_grouped_kernel runs all dW products of
// a W op as one persistent launch over the union of their tiles.  Operands may be K-major or MN-major (SWIZZLE_128B
// canonical layouts, selected by the instruction descriptor's major bits), so
// dX = dY W and dW = dY^T X read the stored activations without transposes.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../../include/adaptra.h"
#include "../prof.h"
#include "../util.h"
#include "common.cuh"
#include "epilogue.cuh"

namespace adaptra {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one SWIZZLE_128B row
// 12 warps: 0..7 epilogue (two warpgroups, two warps per TMEM lane quadrant,
// each owning half of the tile's columns), 8 TMA producer, 9 TMEM allocator +
// MMA issuer, 10..11 idle (they complete the third warpgroup for setmaxnreg).
constexpr int kThreads = 384;
constexpr int kEpiWarps = 8;
constexpr int kWarpProducer = 8, kWarpMma = 9;
constexpr int kWarpSum = 10;  // gemm_tc_grouped_kernel: fused bias-gradient column sums

template <int CG, int BN>
struct TcCfg {
  static constexpr int kBRows = BN / CG;        // B rows held by each CTA
  static constexpr int kStages = CG == 2 ? (BN == 256 ? 5 : 6) : (BN == 256 ? 3 : 5);
  static constexpr int kABytes = BM * BK * 2;    // 16 KB
  static constexpr int kBBytes = kBRows * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;       // two accumulators of 128 lanes x BN columns
  static constexpr int kEpiBytes = kEpiWarps * 8192;  // two 32x32 fp32 staging buffers per epilogue warp
  static constexpr int kSmem = kStages * kStageBytes + kEpiBytes + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int TM = BM * CG;             // tile rows
};

struct TileInfo {
  int m_blocks, n_blocks, Z;
  int k_blocks;  // full K range in BK blocks
};

// TMA-store epilogue: batch offsets of C and of the GELU pre-activation output
// (aux) as (row, col) coordinates of their 2-D tensor maps.
struct EpiTma {
  int on;
  int in_tma;  // RESID / DGELU / DSOFTMAX: the input tile (R or aux) arrives by TMA through tmX
  int c_r1, c_r2, c_q1, c_q2;
  int x_r1, x_r2, x_q1, x_q2;
};

// 32 consecutive bf16 of one row (guarded tail) -> fp32
__device__ __forceinline__ void ld_row32(const bf16* p, int n0, int N, bool vec, float* out) {
  if (vec && n0 + 32 <= N) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) ld_bf16x8(p + j, out + j);
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) out[j] = (n0 + j < N) ? __bfloat162float(p[j]) : 0.f;
  }
}

__device__ __forceinline__ void tile_coords(int t, const TileInfo& ti, int& mb, int& nb, int& z) {
  mb = t % ti.m_blocks;
  int r = t / ti.m_blocks;
  nb = r % ti.n_blocks;
  z = r / ti.n_blocks;
}

// Work units of a launch: one tile each, or (MC: 2x2 clusters of CTA pairs)
// one pair of N-adjacent tiles per cluster, pair pp of the cluster taking
// tile nb = 2 nbp + pp (both need the same A rows, fetched once, multicast).
template <int MC>
__device__ __forceinline__ int n_units(const TileInfo& ti) {
  return MC ? ti.m_blocks * (ti.n_blocks / 2) * ti.Z : ti.m_blocks * ti.n_blocks * ti.Z;
}
template <int MC>
__device__ __forceinline__ void unit_coords(int u, const TileInfo& ti, int pp, int& mb, int& nb, int& z) {
  if (!MC) {
    tile_coords(u, ti, mb, nb, z);
    return;
  }
  const int half = ti.n_blocks / 2;
  mb = u % ti.m_blocks;
  const int r = u / ti.m_blocks;
  nb = 2 * (r % half) + pp;
  z = r / half;
}

// K-block range of a tile (causal variants restrict it), and whether it is skipped.
template <int TM, int BN>
__device__ __forceinline__ bool tile_range(const adaptra_gemm_desc_t& g, const TileInfo& ti, int mb, int nb,
                                           int& kb0, int& kb1) {
  kb0 = 0;
  kb1 = ti.k_blocks;
  if (g.causal == ADAPTRA_CAUSAL_TILE) {
    if (nb * BN > mb * TM + TM - 1) return false;
  } else if (g.causal == ADAPTRA_CAUSAL_KEND) {
    int kend = min(g.K, mb * TM + TM);
    kb1 = (kend + BK - 1) / BK;
  } else if (g.causal == ADAPTRA_CAUSAL_KSTART) {
    kb0 = (mb * TM) / BK;
  }
  return kb1 > kb0;
}

// ---------------------------------------------------------------- epilogue
// Runs in warps 0..7 of every CTA.  Rows of this CTA: tile row0 + rank*128;
// warp w drains lane quadrant w % 4, columns [(w / 4) BN/2, (w / 4 + 1) BN/2).
template <int CG, int BN, int MC>
__device__ __forceinline__ void epilogue_loop(const adaptra_gemm_desc_t& g, const TileInfo& ti, const EpiTma& et,
                                              const CUtensorMap* tmC, const CUtensorMap* tmX, int vec_ok,
                                              uint8_t* sEpi, uint32_t tmem_base, uint64_t* tfull, uint64_t* tempty,
                                              uint64_t* inbar, int warp, int lane, int cid, int ncl, int rank, int pp,
                                              int leader) {
  constexpr int TM = TcCfg<CG, BN>::TM;
  const int n_tiles = n_units<MC>(ti);
  const int quad = warp & 3;  // TMEM lane quadrant this warp may access
  const int co = (warp >> 2) * (BN / 2);  // first column of this warp's half
  constexpr int NC = BN / 64;            // 32-column chunks per warp
  uint8_t* stg = sEpi + warp * 8192;
  int sbuf = 0;
  int acc = 0;
  uint32_t acc_phase = 0;
  uint32_t in_phase = 0;
  // With in_tma the warp's 8 KB staging holds the input tile's NC chunks
  // (2 KB each, bf16, SWIZZLE_64B = the bf16 output staging layout); each
  // chunk's output is written over its input and TMA-stored from there.  No
  // global load is then in flight at the fence.proxy.async of a chunk (it
  // compiles to MEMBAR.ALL.CTA, which would wait for it).
  const bool f32o = (g.epi == ADAPTRA_EPI_ACC_F32 || g.epi == ADAPTRA_EPI_STORE_F32);
  const bool has_in = (g.epi == ADAPTRA_EPI_RESID || g.epi == ADAPTRA_EPI_DGELU || g.epi == ADAPTRA_EPI_DSOFTMAX ||
                       g.epi == ADAPTRA_EPI_STORE_ROWDOT);
  for (int t = cid; t < n_tiles; t += ncl) {
    int mb, nb, z, kb0, kb1;
    unit_coords<MC>(t, ti, pp, mb, nb, z);
    if (!tile_range<TM, BN>(g, ti, mb, nb, kb0, kb1)) continue;
    EpiCtx e = make_epi<bf16>(g, z);
    const int rbase = mb * TM + rank * BM + quad * 32;
    const int m = rbase + lane;
    const bool row_ok = m < e.M;
    const int z1 = z / g.zdiv, z2 = z % g.zdiv;
    const int crow = z1 * et.c_r1 + z2 * et.c_r2 + rbase;
    const int ccol = z1 * et.c_q1 + z2 * et.c_q2 + nb * BN + co;
    const int xrow = z1 * et.x_r1 + z2 * et.x_r2 + rbase;
    const int xcol = z1 * et.x_q1 + z2 * et.x_q2 + nb * BN + co;
    const bool in_tma = has_in && et.in_tma && et.on == 1;
    const bf16* in_row = nullptr;
    if (has_in && row_ok && !in_tma)
      in_row = g.epi == ADAPTRA_EPI_RESID ? (const bf16*)e.R + (long)m * e.ldr : (const bf16*)e.aux + (long)m * e.ldaux;
    float nxt[32];
    if (in_row) ld_row32(in_row + nb * BN + co, nb * BN + co, e.N, vec_ok, nxt);
    if (in_tma && lane == 0) {
      bulk_wait_read<0>();  // the previous tile's stores have read the staging
      mbar_arrive_expect_tx(inbar, NC * 2048);
#pragma unroll
      for (int c = 0; c < NC; ++c) tma_load_2d(stg + c * 2048, tmX, inbar, xcol + c * 32, xrow);
    }
    const float Dm = (g.epi == ADAPTRA_EPI_DSOFTMAX && row_ok) ? e.rowv[m] : 0.f;
    float rdot = 0.f;  // EPI_STORE_ROWDOT: this warp's 128 columns are one head
    mbar_wait(&tfull[acc], acc_phase);
    tc_fence_after();
    const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN + co;
    uint32_t r[32];
    tmem_ld32(tbase, r);  // chunk 0; chunk c+1 is requested while chunk c is processed
#pragma unroll 1
    for (int c = 0; c < NC; ++c) {
      const int n0 = nb * BN + co + c * 32;
      tmem_ld_wait_regs(r);
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
      if (c + 1 < NC) tmem_ld32(tbase + (c + 1) * 32, r);
      float in[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) in[j] = nxt[j];
      if (in_row && c + 1 < NC && n0 + 32 < e.N) ld_row32(in_row + n0 + 32, n0 + 32, e.N, vec_ok, nxt);
      if (n0 >= e.N) continue;
      if (et.on == 2) continue;  // diagnostic: accumulator drained, no epilogue work
      if (!et.on) {
        if (vec_ok && row_ok && n0 + 32 <= e.N)
          epi_row32_bf16_fast(e, m, n0, v);
        else
          epi_row<bf16, 32>(e, m, n0, v);
        continue;
      }
      float bv[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) bv[j] = 0.f;
      if (e.bias && (g.epi == ADAPTRA_EPI_STORE || g.epi == ADAPTRA_EPI_GELU || g.epi == ADAPTRA_EPI_RESID)) {
        if (vec_ok && n0 + 32 <= e.N) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 b4 = *reinterpret_cast<const float4*>(e.bias + n0 + j);
            bv[j] = b4.x; bv[j + 1] = b4.y; bv[j + 2] = b4.z; bv[j + 3] = b4.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) bv[j] = (n0 + j < e.N) ? e.bias[n0 + j] : 0.f;
        }
      }
      uint8_t* sb;
      if (in_tma) {
        if (c == 0) mbar_wait(inbar, in_phase);
        sb = stg + c * 2048;
        const uint8_t* irow = sb + lane * 64;
#pragma unroll
        for (int j = 0; j < 4; ++j) ld_bf16x8((const bf16*)(irow + ((j ^ ((lane >> 1) & 3)) << 4)), in + 8 * j);
      } else {
        // wait until this staging buffer's previous TMA store has read it
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
        sb = stg + sbuf * 4096;
        sbuf ^= 1;
      }
      switch (g.epi) {
        case ADAPTRA_EPI_STORE:
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = e.alpha * v[j] + bv[j];
          break;
        case ADAPTRA_EPI_GELU: {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += bv[j];
          uint8_t* xrow = sb + 2048 + lane * 64;
#pragma unroll
          for (int j = 0; j < 4; ++j) st_bf16x8((bf16*)(xrow + ((j ^ ((lane >> 1) & 3)) << 4)), v + 8 * j);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = gelu_fast(__bfloat162float(__float2bfloat16_rn(v[j])));
        } break;
        case ADAPTRA_EPI_RESID:
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += bv[j] + in[j];
          break;
        case ADAPTRA_EPI_DGELU:
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] *= gelu_grad_fast(in[j]);
          break;
        case ADAPTRA_EPI_DSOFTMAX:
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = in[j] * (v[j] - Dm) * e.alpha;
          break;
        case ADAPTRA_EPI_STORE_ROWDOT:
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            v[j] = __bfloat162float(__float2bfloat16_rn(v[j]));  // the stored dO
            rdot = fmaf(v[j], in[j], rdot);
          }
          break;
        default:  // ACC_F32, STORE_F32
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] *= e.alpha;
          break;
      }
      // staging layout = TMA SWIZZLE_128B (fp32, 128 B rows) / SWIZZLE_64B (bf16,
      // 64 B rows): 16 B chunk k of row r at chunk k ^ f(r) -> conflict-free
      if (f32o) {
        uint8_t* frow = sb + lane * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<float4*>(frow + ((j ^ (lane & 7)) << 4)) =
              make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      } else {
        uint8_t* crow_s = sb + lane * 64;
#pragma unroll
        for (int j = 0; j < 4; ++j) st_bf16x8((bf16*)(crow_s + ((j ^ ((lane >> 1) & 3)) << 4)), v + 8 * j);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (et.on == 3) continue;  // diagnostic: full epilogue except the TMA store itself
      if (lane == 0) {
        if (g.epi == ADAPTRA_EPI_ACC_F32)
          tma_reduce_add_2d(tmC, sb, ccol + c * 32, crow);
        else
          tma_store_2d(tmC, sb, ccol + c * 32, crow);
        if (g.epi == ADAPTRA_EPI_GELU) tma_store_2d(tmX, sb + 2048, xcol + c * 32, xrow);
        bulk_commit();
      }
    }
    if (in_tma) in_phase ^= 1;
    if (g.epi == ADAPTRA_EPI_STORE_ROWDOT && row_ok && et.on == 1) {
      const int Tn = (int)g.rowv_1, Hn = (int)g.rowv_2;
      const int head = (nb * BN + co) / 128, sq = m / Tn, t = m - sq * Tn;
      const_cast<float*>(g.rowv)[((size_t)sq * Hn + head) * Tn + t] = rdot;
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if (CG == 1)
        mbar_arrive(&tempty[acc]);
      else
        mbar_arrive_remote(&tempty[acc], leader);  // the pair leader reuses the accumulator
    }
    if (++acc == 2) {
      acc = 0;
      acc_phase ^= 1;
    }
  }
  if (lane == 0) bulk_wait<0>();
}

// ---------------------------------------------------------------- kernel
template <int CG, int BN, int AMN, int BMN, int MC>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmX,
                   const adaptra_gemm_desc_t g, const TileInfo ti, int vec_ok, const EpiTma et) {
  using Cfg = TcCfg<CG, BN>;
  constexpr int TM = Cfg::TM;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + Cfg::kStages * Cfg::kABytes;
  uint8_t* sEpi = smem + Cfg::kStages * Cfg::kStageBytes;
  uint64_t* full = (uint64_t*)(smem + Cfg::kStages * Cfg::kStageBytes + Cfg::kEpiBytes);
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* tfull = empty + Cfg::kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* inbar = tempty + 2;  // [kEpiWarps] epilogue input tiles (in_tma)
  uint32_t* tmem_slot = (uint32_t*)(inbar + kEpiWarps);

  static_assert(!MC || (CG == 2 && AMN == 0), "multicast: CTA pairs, K-major A");
  constexpr int CL = MC ? 4 : CG;  // CTAs per cluster
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int crank = CG == 2 ? (int)cluster_ctarank() : 0;
  const int rank = crank & 1;          // CTA within its pair
  const int pp = MC ? crank >> 1 : 0;  // pair within the cluster
  const int leader = crank & ~1;       // cluster rank of this pair's leader
  const int cid = blockIdx.x / CL;
  const int ncl = gridDim.x / CL;
  const int n_tiles = n_units<MC>(ti);

  if (warp == kWarpProducer && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < Cfg::kStages; ++s) {
      mbar_init(&full[s], 1);
      // MC: a stage is refilled only when the MMAs of both pairs are done
      // with it (the A halves land in both pairs' shared memory)
      mbar_init(&empty[s], MC ? 2 : 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarps * CG);
    }
    for (int w = 0; w < kEpiWarps; ++w) mbar_init(&inbar[w], 1);
    fence_barrier_init();
  }
  if (warp == kWarpMma) {
    if (CG == 1)
      tmem_alloc(tmem_slot, Cfg::kTmemCols);
    else
      tmem_alloc2(tmem_slot, Cfg::kTmemCols);
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // register budget: the epilogue warpgroups grow, the producer/MMA warpgroup
  // shrinks (setmaxnreg executed uniformly per warpgroup at the top of its branch)
  if (warp >= kEpiWarps) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 40;" ::: "memory");
  if (warp == kWarpProducer) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < n_tiles; t += ncl) {
        int mb, nb, z, kb0, kb1;
        unit_coords<MC>(t, ti, pp, mb, nb, z);
        if (!tile_range<TM, BN>(g, ti, mb, nb, kb0, kb1)) continue;
        const int z1 = z / g.zdiv, z2 = z % g.zdiv;
        const int a_r = (int)(z1 * g.a_row1 + z2 * g.a_row2), a_c = (int)(z1 * g.a_col1 + z2 * g.a_col2);
        const int b_r = (int)(z1 * g.b_row1 + z2 * g.b_row2), b_c = (int)(z1 * g.b_col1 + z2 * g.b_col2);
        const int m0 = mb * TM + rank * BM, n0 = nb * BN + rank * Cfg::kBRows;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], Cfg::kStageBytes * CG);
          uint8_t* a_dst = sA + stage * Cfg::kABytes;
          uint8_t* b_dst = sB + stage * Cfg::kBBytes;
          const int k0 = kb * BK;
          if (CG == 1) {
            if (AMN == 0) {
              tma_load_2d(a_dst, &tmA, &full[stage], a_c + k0, a_r + m0);
            } else {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j)
                tma_load_2d(a_dst + j * (BK * 128), &tmA, &full[stage], a_c + m0 + 64 * j, a_r + k0);
            }
            if (BMN == 0) {
              tma_load_2d(b_dst, &tmB, &full[stage], b_c + k0, b_r + n0);
            } else {
#pragma unroll
              for (int j = 0; j < Cfg::kBRows / 64; ++j)
                tma_load_2d(b_dst + j * (BK * 128), &tmB, &full[stage], b_c + n0 + 64 * j, b_r + k0);
            }
          } else {
            if (MC) {
              // this CTA fetches half of its A rows (box BM/2) for itself and
              // its counterpart in the other pair, which fetches the other half
              const uint16_t mask = (uint16_t)((1u << crank) | (1u << (crank ^ 2)));
              tma_load_2d_2sm_mc(a_dst + pp * (BM / 2) * 128, &tmA, &full[stage], a_c + k0, a_r + m0 + pp * (BM / 2),
                                 mask);
            } else if (AMN == 0) {
              tma_load_2d_2sm(a_dst, &tmA, &full[stage], a_c + k0, a_r + m0);
            } else {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j)
                tma_load_2d_2sm(a_dst + j * (BK * 128), &tmA, &full[stage], a_c + m0 + 64 * j, a_r + k0);
            }
            if (BMN == 0) {
              tma_load_2d_2sm(b_dst, &tmB, &full[stage], b_c + k0, b_r + n0);
            } else {
#pragma unroll
              for (int j = 0; j < Cfg::kBRows / 64; ++j)
                tma_load_2d_2sm(b_dst + j * (BK * 128), &tmB, &full[stage], b_c + n0 + 64 * j, b_r + k0);
            }
          }
          if (++stage == Cfg::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == kWarpMma) {
    // ===================== MMA issuer (leader CTA) =====================
    // Instruction descriptor, kind::f16: D f32 (bit 4), A bf16 (bits 7-9 = 1),
    // B bf16 (bits 10-12 = 1), A/B major (bits 15/16), N>>3 (17-22), M>>4 (24-28).
    if (rank == 0) {
      const uint16_t empty_mask = MC ? 0xF : 3, pair_mask = (uint16_t)(3u << (2 * pp));
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)AMN << 15) | ((uint32_t)BMN << 16) |
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cid; t < n_tiles; t += ncl) {
        int mb, nb, z, kb0, kb1;
        unit_coords<MC>(t, ti, pp, mb, nb, z);
        if (!tile_range<TM, BN>(g, ti, mb, nb, kb0, kb1)) continue;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(sA + stage * Cfg::kABytes);
            const uint32_t b_addr = smem_u32(sB + stage * Cfg::kBBytes);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              // K-major: advance 16 elements = 32 B inside the swizzled row; SBO = 8 rows x 128 B.
              // MN-major: advance 16 K-rows = 2 KB; LBO = one 64-wide MN chunk (BK x 128 B), SBO = 8 rows.
              uint64_t ad = AMN == 0 ? umma_desc_sw128(a_addr + k * 32, 16, 1024)
                                     : umma_desc_sw128(a_addr + k * 2048, BK * 128, 1024);
              uint64_t bd = BMN == 0 ? umma_desc_sw128(b_addr + k * 32, 16, 1024)
                                     : umma_desc_sw128(b_addr + k * 2048, BK * 128, 1024);
              if (CG == 1)
                tc_mma_f16(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
              else
                tc_mma_f16_2sm(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            }
            if (CG == 1)
              tc_commit(&empty[stage]);
            else
              tc_commit_2sm_mc(&empty[stage], empty_mask);
          }
          __syncwarp();
          if (++stage == Cfg::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) {
          if (CG == 1)
            tc_commit(&tfull[acc]);
          else
            tc_commit_2sm_mc(&tfull[acc], pair_mask);
        }
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory");
    epilogue_loop<CG, BN, MC>(g, ti, et, &tmC, &tmX, vec_ok, sEpi, tmem_base, tfull, tempty, &inbar[warp], warp, lane,
                              cid, ncl, rank, pp, leader);
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  if (warp == kWarpMma) {
    if (CG == 1)
      tmem_dealloc(tmem_base, Cfg::kTmemCols);
    else
      tmem_dealloc2(tmem_base, Cfg::kTmemCols);
  }
}

// ------------------------------------------------------------------ host side

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)p;
  });
  return fn;
}

// 2-D map over a [rows, cols] row-major matrix with leading dimension ld
// (bf16 operands: SWIZZLE_128B boxes; epilogue outputs: unswizzled 32x32 boxes).
static int make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_c,
                    int box_r, bool f32 = false, int swz = 128) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return set_error(ADAPTRA_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * (f32 ? 4 : 2))};
  cuuint32_t box[2] = {(cuuint32_t)box_c, (cuuint32_t)box_r};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                              : (swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE),
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(ADAPTRA_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return ADAPTRA_OK;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// SMs a persistent GEMM launch may use (adaptra_set_tuning
// ADAPTRA_TUNE_GEMM_SMS; 0 = all).  With several stages sharing a GPU the
// other stages' kernels fill the rest, and each CTA runs more tiles, so its
// prologue and its last epilogue are paid over more work.
std::atomic<int> g_gemm_sms{0};
extern std::atomic<int> g_attn_sms;  // attn_tc.cu
static int gemm_sms() {
  const int cap = g_gemm_sms.load(std::memory_order_relaxed);
  const int n = num_sms();
  return (cap > 0 && cap < n) ? cap : n;
}

template <int CG, int BN, int AMN, int BMN, int MC = 0>
static int launch_tc(const adaptra_gemm_desc_t& g, cudaStream_t st) {
  using Cfg = TcCfg<CG, BN>;
  CUtensorMap ma, mbm;
  int rc;
  if (AMN == 0)
    rc = make_map(&ma, g.A, g.a_rows, g.a_cols, g.lda, BK, MC ? BM / 2 : BM);
  else
    rc = make_map(&ma, g.A, g.a_rows, g.a_cols, g.lda, 64, BK);
  if (rc) return rc;
  if (BMN == 0)
    rc = make_map(&mbm, g.B, g.b_rows, g.b_cols, g.ldb, BK, Cfg::kBRows);
  else
    rc = make_map(&mbm, g.B, g.b_rows, g.b_cols, g.ldb, 64, BK);
  if (rc) return rc;
  TileInfo ti;
  ti.m_blocks = (g.M + Cfg::TM - 1) / Cfg::TM;
  ti.n_blocks = (g.N + BN - 1) / BN;
  ti.Z = g.Z;
  ti.k_blocks = (g.K + BK - 1) / BK;
  const int n_tiles = MC ? ti.m_blocks * (ti.n_blocks / 2) * ti.Z : ti.m_blocks * ti.n_blocks * ti.Z;
  auto kern = gemm_tc_kernel<CG, BN, AMN, BMN, MC>;
  static std::atomic<unsigned> attr_mask{0};  // per device; stage threads may race here
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_mask.load(std::memory_order_acquire) & (1u << dev))) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    attr_mask.fetch_or(1u << dev, std::memory_order_release);
  }
  bool f32out = (g.epi == ADAPTRA_EPI_ACC_F32 || g.epi == ADAPTRA_EPI_STORE_F32);
  int vec_ok = (g.ldc % (f32out ? 4 : 8) == 0) && ((uintptr_t)g.C % 16 == 0) &&
               (!g.aux || (g.ldaux % 8 == 0 && (uintptr_t)g.aux % 16 == 0)) &&
               (!g.R || (g.ldr % 8 == 0 && (uintptr_t)g.R % 16 == 0)) && ((uintptr_t)g.bias % 16 == 0) &&
               (g.c_1 % 8 == 0) && (g.c_2 % 8 == 0) && (g.aux_1 % 8 == 0) && (g.aux_2 % 8 == 0);
  constexpr int CL = MC ? 4 : CG;
  const int slots = std::max(1, gemm_sms() / CL);
  int grid = (n_tiles < slots ? n_tiles : slots) * CL;
  if (grid < 1) return ADAPTRA_OK;
  // TMA-store epilogue when C (and the GELU aux output) decompose into 2-D
  // coordinates and live on this device (a peer mailbox is written with
  // plain stores).
  EpiTma et{};
  CUtensorMap mc, mx;
  memset(&mc, 0, sizeof(mc));
  memset(&mx, 0, sizeof(mx));
  {
    const int64_t esz = f32out ? 4 : 2;
    auto decomp = [&](int64_t o1, int64_t o2, int64_t ld, int& r1, int& r2, int& q1, int& q2, int64_t& rows,
                      int64_t& cols) {
      r1 = (int)(o1 / ld); q1 = (int)(o1 % ld);
      r2 = (int)(o2 / ld); q2 = (int)(o2 % ld);
      const int64_t z1m = (g.Z - 1) / g.zdiv, z2m = g.Z > 1 ? (g.zdiv - 1) : 0;
      cols = z1m * q1 + z2m * q2 + g.N;
      rows = z1m * r1 + z2m * r2 + g.M;
      return cols <= ld || g.Z == 1;
    };
    bool ok = vec_ok && ((uintptr_t)g.C % 16 == 0) && (g.ldc * esz) % 16 == 0;
    if (ok && g.epi == ADAPTRA_EPI_RESID) {
      cudaPointerAttributes pa;
      int dev = 0;
      cudaGetDevice(&dev);
      ok = cudaPointerGetAttributes(&pa, g.C) == cudaSuccess && pa.type == cudaMemoryTypeDevice && pa.device == dev;
      cudaGetLastError();
    }
    int64_t rows = 0, cols = 0;
    if (ok) ok = decomp(g.c_1, g.c_2, g.ldc, et.c_r1, et.c_r2, et.c_q1, et.c_q2, rows, cols);
    if (ok)
      ok = make_map(&mc, g.C, rows, g.Z == 1 ? g.N : cols, g.ldc, 32, 32, f32out, f32out ? 128 : 64) == ADAPTRA_OK;
    if (ok && g.epi == ADAPTRA_EPI_GELU) {
      int64_t xr = 0, xc = 0;
      ok = g.aux && ((uintptr_t)g.aux % 16 == 0) &&
           decomp(g.aux_1, g.aux_2, g.ldaux, et.x_r1, et.x_r2, et.x_q1, et.x_q2, xr, xc) &&
           make_map(&mx, g.aux, xr, g.Z == 1 ? g.N : xc, g.ldaux, 32, 32, false, 64) == ADAPTRA_OK;
    }
    if (ok && (g.epi == ADAPTRA_EPI_DGELU || g.epi == ADAPTRA_EPI_DSOFTMAX || g.epi == ADAPTRA_EPI_STORE_ROWDOT) &&
        g.aux && (uintptr_t)g.aux % 16 == 0 &&
        (g.ldaux * 2) % 16 == 0) {
      int64_t xr = 0, xc = 0;
      et.in_tma = decomp(g.aux_1, g.aux_2, g.ldaux, et.x_r1, et.x_r2, et.x_q1, et.x_q2, xr, xc) &&
                  make_map(&mx, g.aux, xr, g.Z == 1 ? g.N : xc, g.ldaux, 32, 32, false, 64) == ADAPTRA_OK;
    } else if (ok && g.epi == ADAPTRA_EPI_RESID && g.R && (uintptr_t)g.R % 16 == 0 && (g.ldr * 2) % 16 == 0 &&
               g.Z == 1) {
      et.x_r1 = et.x_r2 = et.x_q1 = et.x_q2 = 0;
      et.in_tma = make_map(&mx, g.R, g.M, g.N, g.ldr, 32, 32, false, 64) == ADAPTRA_OK;
    }
    static const bool no_in_tma = getenv("ADAPTRA_EPI_IN_LDG") != nullptr;  // timing comparison only
    if (no_in_tma && g.epi != ADAPTRA_EPI_STORE_ROWDOT) et.in_tma = 0;
    et.on = ok ? 1 : 0;
    // timing experiments only: 1 = skip all epilogue work, 2 = skip the TMA store
    static const int diag = getenv("ADAPTRA_DIAG_NOEPI") ? atoi(getenv("ADAPTRA_DIAG_NOEPI")) : 0;
    if (g.epi == ADAPTRA_EPI_STORE_ROWDOT && !(et.on == 1 && et.in_tma && CG == 2 && BN == 256)) {
      cudaGetLastError();
      return set_error(ADAPTRA_EINVAL, "STORE_ROWDOT needs the TMA epilogue of the 2-CTA 256-wide path");
    }
    if (diag == 1 && ok) et.on = 2;
    if (diag == 2 && ok) et.on = 3;
    cudaGetLastError();
  }
  void* pb = prof_on() ? prof_begin(st) : nullptr;
  if (CG == 1) {
    kern<<<grid, kThreads, Cfg::kSmem, st>>>(ma, mbm, mc, mx, g, ti, vec_ok, et);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Cfg::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, ma, mbm, mc, mx, g, ti, vec_ok, et);
  }
  count_launch();
  if (pb) {
    // algorithmic FLOPs: 2MNK per batch; causal variants count the lower half (R28)
    double fl = 2.0 * g.M * (double)g.N * g.K * g.Z * (g.causal ? 0.5 : 1.0);
    bool f32o = (g.epi == ADAPTRA_EPI_ACC_F32 || g.epi == ADAPTRA_EPI_STORE_F32);
    double by = 2.0 * ((double)g.M * g.K + (double)g.N * g.K) * g.Z + (f32o ? 4.0 : 2.0) * g.M * (double)g.N * g.Z;
    prof_end(pb, st, g.Z == 1 ? PROF_GEMM_TC : PROF_GEMM_ATTN, fl, by);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ADAPTRA_ECUDA, std::string("gemm_tc launch: ") + cudaGetErrorString(e));
  return ADAPTRA_OK;
}

// ------------------------------------------------------------------ grouped dW
// All weight-gradient products of a W op (dW += X^T dY for every
// linear layer of the stage) are independent, so they run as one persistent
// launch over the union of their tiles instead of one launch each: the waves
// are filled across problems and only the launch's last tiles expose an
// epilogue.  Specialised to what W needs: CTA pairs, 256 x 256 tiles, both
// operands MN-major, fp32 TMA reduce-add into the gradient.  Each tile runs
// the same MMA sequence and reduce-add as in gemm_tc_kernel, so the result is
// the same bit for bit.
constexpr int kMaxGroup = 24;
// Up to kMaxSeg K segments per product (W of up to kMaxSeg slots: segment s
// covers K blocks [s*k_seg, (s+1)*k_seg) from its own A / B tensor maps).
constexpr int kMaxSeg = 4;
struct GroupArgs {
  CUtensorMap tmA[kMaxSeg][kMaxGroup], tmB[kMaxSeg][kMaxGroup], tmC[kMaxGroup];
  int n, total_tiles;
  int tile_start[kMaxGroup + 1];
  int m_blocks[kMaxGroup], k_blocks[kMaxGroup], k_seg[kMaxGroup], N[kMaxGroup], M[kMaxGroup];
  float alpha[kMaxGroup];
  float* dbias[kMaxGroup];  // db += column sums of A (= dY) over K, or NULL
  int sum_mode;             // 1: the column-sum warp runs (some dbias set)
};
static_assert(sizeof(GroupArgs) <= 32000, "grouped GEMM kernel parameter too large");

__device__ __forceinline__ void group_tile(const GroupArgs& ga, int t, int TM_, int& q, int& mb, int& nb) {
  q = 0;
  while (q + 1 < ga.n && t >= ga.tile_start[q + 1]) ++q;
  const int lt = t - ga.tile_start[q];
  mb = lt % ga.m_blocks[q];
  nb = lt / ga.m_blocks[q];
  (void)TM_;
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1) gemm_tc_grouped_kernel(const __grid_constant__ GroupArgs ga) {
  constexpr int CG = 2;
  using Cfg = TcCfg<CG, BN>;
  constexpr int TM = Cfg::TM;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + Cfg::kStages * Cfg::kABytes;
  uint8_t* sEpi = smem + Cfg::kStages * Cfg::kStageBytes;
  uint64_t* full = (uint64_t*)(smem + Cfg::kStages * Cfg::kStageBytes + Cfg::kEpiBytes);
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* tfull = empty + Cfg::kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2 + kEpiWarps;  // [kStages] stage landed, for the column-sum warp
  uint32_t* tmem_slot = (uint32_t*)(sfull + Cfg::kStages);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int rank = (int)cluster_ctarank();
  const int cid = blockIdx.x / 2, ncl = gridDim.x / 2;

  if (warp == kWarpProducer && lane == 0) {
    for (int s = 0; s < Cfg::kStages; ++s) {
      mbar_init(&full[s], 1);
      // the pair's MMA commit (+ this CTA's column-sum warp when it runs)
      mbar_init(&empty[s], ga.sum_mode ? 2 : 1);
      mbar_init(&sfull[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarps * CG);
    }
    fence_barrier_init();
  }
  if (warp == kWarpMma) tmem_alloc2(tmem_slot, Cfg::kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp >= kEpiWarps) {
  // 56, not 40: the column-sum warp's loop spills at 40 (the epilogue's 208
  // still fits: 128 x 112 released >= 256 x 40 taken)
  asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
  if (warp == kWarpProducer) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < ga.total_tiles; t += ncl) {
        int q, mb, nb;
        group_tile(ga, t, TM, q, mb, nb);
        const int m0 = mb * TM + rank * BM, n0 = nb * BN + rank * Cfg::kBRows;
        for (int kb = 0; kb < ga.k_blocks[q]; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], Cfg::kStageBytes * CG);
          uint8_t* a_dst = sA + stage * Cfg::kABytes;
          uint8_t* b_dst = sB + stage * Cfg::kBBytes;
          const int seg = kb / ga.k_seg[q];
          const int k0 = (kb - seg * ga.k_seg[q]) * BK;
          const CUtensorMap* mA = &ga.tmA[seg][q];
          const CUtensorMap* mB = &ga.tmB[seg][q];
#pragma unroll
          for (int j = 0; j < BM / 64; ++j)
            tma_load_2d_2sm(a_dst + j * (BK * 128), mA, &full[stage], m0 + 64 * j, k0);
#pragma unroll
          for (int j = 0; j < Cfg::kBRows / 64; ++j)
            tma_load_2d_2sm(b_dst + j * (BK * 128), mB, &full[stage], n0 + 64 * j, k0);
          if (++stage == Cfg::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == kWarpMma) {
    if (rank == 0) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cid; t < ga.total_tiles; t += ncl) {
        int q, mb, nb;
        group_tile(ga, t, TM, q, mb, nb);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        const int kb1 = ga.k_blocks[q];
        for (int kb = 0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(sA + stage * Cfg::kABytes);
            const uint32_t b_addr = smem_u32(sB + stage * Cfg::kBBytes);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              tc_mma_f16_2sm(d_tmem, umma_desc_sw128(a_addr + k * 2048, BK * 128, 1024),
                             umma_desc_sw128(b_addr + k * 2048, BK * 128, 1024), idesc, (kb > 0 || k > 0) ? 1u : 0u);
            tc_commit_2sm_mc(&empty[stage]);
            // the stage's MMAs done: each CTA's column-sum warp may read its
            // half (a hardware arrive on both CTAs -- a thread-issued
            // cluster-scope arrive per stage throttled the whole pipeline)
            if (ga.sum_mode) tc_commit_2sm_mc(&sfull[stage]);
          }
          __syncwarp();
          if (++stage == Cfg::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) tc_commit_2sm_mc(&tfull[acc]);
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp == kWarpSum) {
    // Bias gradients fused into the dW products (db += sum_t dY):
    // A is dY, MN-major, so the tiles of column block 0 see every token of
    // their 256 output features.  This CTA's half (128 features, two 64-wide
    // SWIZZLE_128B boxes of BK tokens) is summed from shared memory once the
    // stage's MMAs are done (sfull, committed by the MMA issuer to both CTAs)
    // and before the producer may refill it (empty counts this warp): lane l
    // owns 4 features of box l / 16; per-stage partials, then a running sum
    // -- a fixed order, so the result is deterministic.  Tiles of other
    // column blocks only pass the stage on.
    const int fb = lane >> 4, f4 = (lane & 15) * 4;
    const uint32_t chunk = (uint32_t)(f4 >> 3), hoff = (uint32_t)(f4 & 7) * 2;
    int stage = 0;
    uint32_t phase = 0;
    for (int t = ga.sum_mode ? cid : ga.total_tiles; t < ga.total_tiles; t += ncl) {
      int q, mb, nb;
      group_tile(ga, t, TM, q, mb, nb);
      const bool on = nb == 0 && ga.dbias[q] != nullptr;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      for (int kb = 0; kb < ga.k_blocks[q]; ++kb) {
        mbar_wait(&sfull[stage], phase);
        if (on) {
          const uint32_t box = smem_u32(sA + stage * Cfg::kABytes) + fb * (BK * 128);
          float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
#pragma unroll 16
          for (int k = 0; k < BK; ++k) {
            uint32_t x, y;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];"
                         : "=r"(x), "=r"(y)
                         : "r"(box + k * 128 + (((chunk ^ (uint32_t)(k & 7)) << 4) | hoff)));
            p0 += __uint_as_float(x << 16);
            p1 += __uint_as_float(x & 0xffff0000u);
            p2 += __uint_as_float(y << 16);
            p3 += __uint_as_float(y & 0xffff0000u);
          }
          s0 += p0;
          s1 += p1;
          s2 += p2;
          s3 += p3;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == Cfg::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (on) {
        const int m = mb * TM + rank * BM + fb * 64 + f4;
        float* db = ga.dbias[q] + m;
        const int lim = ga.M[q] - m;
        if (lim > 0) db[0] += s0;
        if (lim > 1) db[1] += s1;
        if (lim > 2) db[2] += s2;
        if (lim > 3) db[3] += s3;
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory");
    // epilogue: fp32 TMA reduce-add of the accumulator (as gemm_tc_kernel's ACC_F32 path)
    const int quad = warp & 3;
    const int co = (warp >> 2) * (BN / 2);
    constexpr int NC = BN / 64;
    uint8_t* stg = sEpi + warp * 8192;
    int sbuf = 0, acc = 0;
    uint32_t acc_phase = 0;
    for (int t = cid; t < ga.total_tiles; t += ncl) {
      int q, mb, nb;
      group_tile(ga, t, TM, q, mb, nb);
      const int crow = mb * TM + rank * BM + quad * 32;
      const int ccol = nb * BN + co;
      const float alpha = ga.alpha[q];
      const int Nq = ga.N[q];
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN + co;
      uint32_t r[32];
      tmem_ld32(tbase, r);
#pragma unroll 1
      for (int c = 0; c < NC; ++c) {
        tmem_ld_wait_regs(r);
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * alpha;
        if (c + 1 < NC) tmem_ld32(tbase + (c + 1) * 32, r);
        if (ccol + c * 32 >= Nq) continue;
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
        uint8_t* sb = stg + sbuf * 4096;
        sbuf ^= 1;
        uint8_t* frow = sb + lane * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<float4*>(frow + ((j ^ (lane & 7)) << 4)) =
              make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_reduce_add_2d(&ga.tmC[q], sb, ccol + c * 32, crow);
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(&tempty[acc], 0);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == kWarpMma) tmem_dealloc2(tmem_base, Cfg::kTmemCols);
}

int gemm_tc(const adaptra_gemm_desc_t& g, cudaStream_t st);

// Grouped dW products (see above).  Falls back to one gemm_tc launch per
// product when a product does not fit the specialisation.
int gemm_tc_grouped(const adaptra_gemm_desc_t* gs, int n, cudaStream_t st, const adaptra_gemm_desc_t* const* more,
                    int n_more, float* const* dbias, bool* fused) {
  if (fused) *fused = false;
  constexpr int BN = 256;
  using Cfg = TcCfg<2, BN>;
  static const bool off = getenv("ADAPTRA_GEMM_GROUPED") && atoi(getenv("ADAPTRA_GEMM_GROUPED")) == 0;
  bool ok = !off && n > 0 && n <= kMaxGroup;
  auto fits = [](const adaptra_gemm_desc_t& g) {
    return g.dtype == ADAPTRA_BF16 && g.Z == 1 && g.epi == ADAPTRA_EPI_ACC_F32 && g.a_mn == 1 && g.b_mn == 1 &&
           !g.causal && g.N >= 2048 && g.M >= 256 && (g.ldc % 4) == 0 && ((uintptr_t)g.C % 16) == 0 &&
           (g.lda * 2) % 16 == 0 && (g.ldb * 2) % 16 == 0 && g.K % BK == 0;
  };
  if (n_more < 0 || n_more > kMaxSeg - 1) return set_error(ADAPTRA_EINVAL, "gemm_tc_grouped: too many K segments");
  for (int i = 0; ok && i < n; ++i) {
    ok = fits(gs[i]);
    for (int m = 0; ok && m < n_more; ++m) {
      const auto& h = more[m][i];
      ok = fits(h) && h.M == gs[i].M && h.N == gs[i].N && h.K == gs[i].K && h.C == gs[i].C && h.ldc == gs[i].ldc &&
           h.alpha == gs[i].alpha;
    }
  }
  if (!ok) {
    for (int i = 0; i < n; ++i) {
      int rc = gemm_tc(gs[i], st);
      for (int m = 0; !rc && m < n_more; ++m) rc = gemm_tc(more[m][i], st);
      if (rc) return rc;
    }
    return ADAPTRA_OK;
  }
  static GroupArgs ga;  // host staging of the kernel parameter (~28 KB); launches are serialised per process
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  memset(&ga, 0, sizeof(ga));
  ga.n = n;
  int tiles = 0;
  double fl = 0;
  for (int i = 0; i < n; ++i) {
    const auto& g = gs[i];
    int rc = make_map(&ga.tmA[0][i], g.A, g.a_rows, g.a_cols, g.lda, 64, BK);
    if (!rc) rc = make_map(&ga.tmB[0][i], g.B, g.b_rows, g.b_cols, g.ldb, 64, BK);
    if (!rc) rc = make_map(&ga.tmC[i], g.C, g.M, g.N, g.ldc, 32, 32, true, 128);
    if (rc) return rc;
    ga.m_blocks[i] = (g.M + Cfg::TM - 1) / Cfg::TM;
    ga.k_blocks[i] = ga.k_seg[i] = g.K / BK;
    ga.N[i] = g.N;
    ga.M[i] = g.M;
    ga.alpha[i] = g.alpha;
    ga.dbias[i] = dbias ? dbias[i] : nullptr;
    if (dbias && dbias[i]) ga.sum_mode = 1;
    ga.tile_start[i] = tiles;
    tiles += ga.m_blocks[i] * ((g.N + BN - 1) / BN);
    fl += 2.0 * g.M * (double)g.N * g.K;
    for (int m = 0; m < n_more; ++m) {
      const auto& h = more[m][i];
      rc = make_map(&ga.tmA[m + 1][i], h.A, h.a_rows, h.a_cols, h.lda, 64, BK);
      if (!rc) rc = make_map(&ga.tmB[m + 1][i], h.B, h.b_rows, h.b_cols, h.ldb, 64, BK);
      if (rc) return rc;
      ga.k_blocks[i] += h.K / BK;
      fl += 2.0 * h.M * (double)h.N * h.K;
    }
  }
  ga.tile_start[n] = tiles;
  ga.total_tiles = tiles;
  auto kern = gemm_tc_grouped_kernel<BN>;
  static std::atomic<unsigned> attr_mask{0};  // per device; stage threads may race here
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_mask.load(std::memory_order_acquire) & (1u << dev))) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    attr_mask.fetch_or(1u << dev, std::memory_order_release);
  }
  const int slots = std::max(1, gemm_sms() / 2);
  const int grid = (tiles < slots ? tiles : slots) * 2;
  void* pb = prof_on() ? prof_begin(st) : nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, ga);
  count_launch();
  if (pb) prof_end(pb, st, PROF_GEMM_TC, fl, 0);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ADAPTRA_ECUDA, std::string("gemm_tc_grouped launch: ") + cudaGetErrorString(e));
  if (fused) *fused = dbias != nullptr;
  return ADAPTRA_OK;
}

int gemm_tc(const adaptra_gemm_desc_t& g, cudaStream_t st) {
  if (g.epi == ADAPTRA_EPI_STORE_ROWDOT &&
      (g.Z != 1 || g.N % 256 || g.N < 2048 || g.M < 256 || g.causal || !g.aux || !g.rowv || g.rowv_1 < 1 ||
       g.rowv_2 < 1))
    return set_error(ADAPTRA_EINVAL, "STORE_ROWDOT: unbatched, N % 256 == 0, N >= 2048, aux and rowv required");
  // BN = 256 for large unbatched N, else 128 (batched attention tiles must not
  // cross a batch boundary: require tile-aligned extents when Z > 1).
  if (g.Z > 1 && (g.M % BM || g.K % BK)) return set_error(ADAPTRA_EINVAL, "batched tc gemm needs M%128==0, K%64==0");
  if ((g.lda * 2) % 16 || (g.ldb * 2) % 16) return set_error(ADAPTRA_EINVAL, "tc gemm needs 16B-aligned rows");
  if (g.Z > 1 && g.N % 128) return set_error(ADAPTRA_EINVAL, "batched tc gemm needs N%128==0");
  // Large unbatched products: CTA pair, 256 x 256 tiles (cta_group::2);
  // otherwise (attention batches, small N) one CTA, 128 x 128 tiles.
  static const int mode = [] {
    const char* v = getenv("ADAPTRA_GEMM_PAIR");
    return v ? atoi(v) : 1;
  }();
  const bool big = (g.Z == 1 && g.N >= 2048 && g.M >= 256 && g.causal == ADAPTRA_CAUSAL_NONE);
  const int key = g.a_mn * 2 + g.b_mn;
  // CTA-pair tile width 256 (default).  256 x 128 tiles (ADAPTRA_GEMM_BN=128)
  // give finer waves over the 74 pairs but were measured 1.3-1.6x slower on
  // every C1 stage shape (profiles/r02_gemm_bn128_vs_bn256.txt): an M = 256,
  // N = 128 MMA moves the same A operand from shared memory for half the
  // FLOPs, so the main loop runs at about half the tensor rate.
  static const int bn_pref = [] {
    const char* v = getenv("ADAPTRA_GEMM_BN");
    return v ? atoi(v) : 256;
  }();
  if (big && mode == 1 && bn_pref == 128 && g.epi != ADAPTRA_EPI_STORE_ROWDOT) {
    switch (key) {
      case 0: return launch_tc<2, 128, 0, 0>(g, st);
      case 1: return launch_tc<2, 128, 0, 1>(g, st);
      case 2: return launch_tc<2, 128, 1, 0>(g, st);
      default: return launch_tc<2, 128, 1, 1>(g, st);
    }
  }
  // 2x2 clusters with the A tile multicast to both CTA pairs
  // ($ADAPTRA_GEMM_MC=1): needs an even number of 256-column tiles, K-major A
  static const bool mc_on = getenv("ADAPTRA_GEMM_MC") && atoi(getenv("ADAPTRA_GEMM_MC")) == 1;
  if (big && mode == 1 && mc_on && g.a_mn == 0 && ((g.N + 255) / 256) % 2 == 0 && g.epi != ADAPTRA_EPI_STORE_ROWDOT) {
    if (g.b_mn == 0) return launch_tc<2, 256, 0, 0, 1>(g, st);
    return launch_tc<2, 256, 0, 1, 1>(g, st);
  }
  if (big && mode == 1) {
    switch (key) {
      case 0: return launch_tc<2, 256, 0, 0>(g, st);
      case 1: return launch_tc<2, 256, 0, 1>(g, st);
      case 2: return launch_tc<2, 256, 1, 0>(g, st);
      default: return launch_tc<2, 256, 1, 1>(g, st);
    }
  }
  if (big) {
    switch (key) {
      case 0: return launch_tc<1, 256, 0, 0>(g, st);
      case 1: return launch_tc<1, 256, 0, 1>(g, st);
      case 2: return launch_tc<1, 256, 1, 0>(g, st);
      default: return launch_tc<1, 256, 1, 1>(g, st);
    }
  }
  switch (key) {
    case 0: return launch_tc<1, 128, 0, 0>(g, st);
    case 1: return launch_tc<1, 128, 0, 1>(g, st);
    case 2: return launch_tc<1, 128, 1, 0>(g, st);
    default: return launch_tc<1, 128, 1, 1>(g, st);
  }
}

}  // namespace adaptra

extern "C" int adaptra_set_tuning(int32_t key, int64_t value) {
  switch (key) {
    case ADAPTRA_TUNE_GEMM_SMS:
      if (value < 0) return adaptra::set_error(ADAPTRA_EINVAL, "set_tuning: SM count must be >= 0");
      adaptra::g_gemm_sms.store((int)value);
      return ADAPTRA_OK;
    case ADAPTRA_TUNE_ATTN_SMS:
      if (value < 0) return adaptra::set_error(ADAPTRA_EINVAL, "set_tuning: SM count must be >= 0");
      adaptra::g_attn_sms.store((int)value);
      return ADAPTRA_OK;
    default:
      return adaptra::set_error(ADAPTRA_EINVAL, "set_tuning: unknown key");
  }
}
