// Stage compute: F / B / W of one pipeline stage (n_layers identical blocks)
// on one microbatch slot, as sequences of the sm_100a kernels.  ZeroBubble
// split: B computes input gradients only and keeps each GEMM's
// output gradient in the slot; W computes all weight gradients later,
// accumulating into fp32 buffers (deferred).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../../include/adaptra.h"
#include "../kernels/kernels.h"
#include "../util.h"

namespace adaptra {
namespace {

struct GB {  // gemm descriptor builder
  adaptra_gemm_desc_t g{};
  explicit GB(int dtype) {
    g.dtype = dtype;
    g.Z = 1;
    g.zdiv = 1;
    g.alpha = 1.f;
  }
  GB& shape(int M, int N, int K) { g.M = M; g.N = N; g.K = K; return *this; }
  GB& batch(int Z, int zdiv) { g.Z = Z; g.zdiv = zdiv; return *this; }
  GB& A(const void* p, long ld, long rows, long cols, int mn = 0, long r1 = 0, long r2 = 0, long c1 = 0, long c2 = 0) {
    g.A = p; g.lda = ld; g.a_rows = rows; g.a_cols = cols; g.a_mn = mn;
    g.a_row1 = r1; g.a_row2 = r2; g.a_col1 = c1; g.a_col2 = c2;
    return *this;
  }
  GB& B(const void* p, long ld, long rows, long cols, int mn = 0, long r1 = 0, long r2 = 0, long c1 = 0, long c2 = 0) {
    g.B = p; g.ldb = ld; g.b_rows = rows; g.b_cols = cols; g.b_mn = mn;
    g.b_row1 = r1; g.b_row2 = r2; g.b_col1 = c1; g.b_col2 = c2;
    return *this;
  }
  GB& C(void* p, long ld, long o1 = 0, long o2 = 0) { g.C = p; g.ldc = ld; g.c_1 = o1; g.c_2 = o2; return *this; }
  GB& epi(int e, float alpha = 1.f) { g.epi = e; g.alpha = alpha; return *this; }
  GB& bias(const float* b) { g.bias = b; return *this; }
  GB& aux(void* p, long ld, long o1 = 0, long o2 = 0) { g.aux = p; g.ldaux = ld; g.aux_1 = o1; g.aux_2 = o2; return *this; }
  GB& res(const void* p, long ld) { g.R = p; g.ldr = ld; return *this; }
  GB& rowv(const float* p, long o1, long o2) { g.rowv = p; g.rowv_1 = o1; g.rowv_2 = o2; return *this; }
  GB& causal(int c) { g.causal = c; return *this; }
  int run(cudaStream_t st) const {
    if (g.M == 0 || g.N == 0) return ADAPTRA_OK;
    return g.dtype == ADAPTRA_BF16 ? gemm_tc(g, st) : gemm_simt(g, st);
  }
};

#define TRY(x)                 \
  do {                         \
    int _rc = (x);             \
    if (_rc) return _rc;       \
  } while (0)

long align256(long v) { return (v + 255) & ~255L; }

}  // namespace

// Byte offsets of the buffers of one slot (per layer) and of the stage work area.
struct SlotLayout {
  long esz;
  // per layer (GPT): xl h1 qkv P o y1 h2 a g dqkv dy1 da dyl dh2 dh1 | f32: mean1 rstd1 mean2 rstd2
  // per layer (MLP): xl a g da dyl
  long xl, h1, qkv, P, o, y1, h2, a, g, dqkv, dy1, da, dyl, dh2, dh1, mean1, rstd1, mean2, rstd2;
  long layer_bytes, fb_layer_bytes, fb_slot_bytes;
  long yL, seed, lpart;  // stage-level (after the per-layer block); lpart: loss partials + ticket
  long slot_bytes;
  // work area
  long w_S, w_dS, w_do, w_D, w_dq, w_cs, w_cnt, cs_floats, cs_tickets, work_bytes;
  bool flash;  // fused tcgen05 attention (bf16, head dim 128)
};

struct adaptra_stage_impl;

}  // namespace adaptra

struct adaptra_stage {
  adaptra_stage_desc_t d;
  int dev = 0;
  adaptra::SlotLayout L;
  long R;  // rows = b*T
  std::vector<const void*> x_in;  // per slot: layer-0 input pointer (mailbox), kept until W
  std::vector<const void*> dy_in;  // per slot: top-layer output gradient pointer
  std::vector<int> fb_of;          // per slot: F->B pool index (-1 if none)
  std::vector<int> fb_free;        // free F->B pool indices (issue order)
};

namespace adaptra {

static bool getenv_materialized() {
  const char* v = getenv("ADAPTRA_ATTN");
  return v && std::string(v) == "materialized";
}

static int compute_layout(const adaptra_stage_desc_t& d, SlotLayout& L) {
  if (d.n_layers < 1 || d.d < 8 || d.d % 8 || d.b < 1 || d.T < 1) return set_error(ADAPTRA_EINVAL, "stage: bad dims");
  if (d.dtype != ADAPTRA_F32 && d.dtype != ADAPTRA_BF16) return set_error(ADAPTRA_EINVAL, "stage: bad dtype");
  const long e = d.dtype == ADAPTRA_BF16 ? 2 : 4;
  const long R = (long)d.b * d.T, D = d.d, F = d.d_ff;
  if (F < 8 || F % 8) return set_error(ADAPTRA_EINVAL, "stage: d_ff must be a multiple of 8");
  L.esz = e;
  long off = 0;
  auto put = [&](long bytes) {
    long o = off;
    off = align256(off + bytes);
    return o;
  };
  L = SlotLayout{};
  L.esz = e;
  if (d.block == ADAPTRA_BLOCK_GPT) {
    if (d.n_heads < 1 || D % d.n_heads) return set_error(ADAPTRA_EINVAL, "stage: d % n_heads != 0");
    long dh = D / d.n_heads;
    if (dh % 8) return set_error(ADAPTRA_EINVAL, "stage: head dim must be a multiple of 8");
    // bf16 runs the tcgen05 path: the fused attention is built for head dim
    // 128 (GPT-2 shapes); other head dims are rejected rather than
    // routed to an untested path (fp32 parity mode takes any multiple of 8)
    if (d.dtype == ADAPTRA_BF16 && (d.T % 128 || dh != 128))
      return set_error(ADAPTRA_EINVAL, "stage bf16: T % 128 == 0 and head dim 128 required");
    long PT = (long)d.b * d.n_heads * d.T * d.T;
    L.xl = put(R * D * e);
    L.h1 = put(R * D * e);
    L.o = put(R * D * e);
    L.y1 = put(R * D * e);
    L.h2 = put(R * D * e);
    L.g = put(R * F * e);
    L.dqkv = put(R * 3 * D * e);
    L.dy1 = put(R * D * e);
    L.da = put(R * F * e);
    L.dyl = put(R * D * e);
    L.dh2 = put(R * D * e);
    L.dh1 = put(R * D * e);
    L.mean1 = put(R * 4);
    L.rstd1 = put(R * 4);
    L.mean2 = put(R * 4);
    L.rstd2 = put(R * 4);
    // F->B pool (freed when B ends): the fused attention keeps only the
    // per-row log-sum-exp instead of the T x T probabilities
    L.flash = d.dtype == ADAPTRA_BF16 && dh == 128 && !getenv_materialized();
    long off_w = off;
    off = 0;
    L.qkv = put(R * 3 * D * e);
    L.P = L.flash ? put((long)d.b * d.n_heads * d.T * 4) : put(PT * e);
    L.a = put(R * F * e);
    L.fb_layer_bytes = off;
    off = off_w;
  } else if (d.block == ADAPTRA_BLOCK_MLP) {
    L.xl = put(R * D * e);
    L.g = put(R * F * e);
    L.da = put(R * F * e);
    L.dyl = put(R * D * e);
    long off_w = off;
    off = 0;
    L.a = put(R * F * e);
    L.fb_layer_bytes = off;
    off = off_w;
  } else {
    return set_error(ADAPTRA_EINVAL, "stage: bad block kind");
  }
  L.layer_bytes = off;
  long tail = L.layer_bytes * d.n_layers;
  L.yL = tail;
  L.seed = align256(L.yL + R * D * e);
  L.lpart = align256(L.seed + R * D * e);
  L.slot_bytes = d.is_last ? align256(L.lpart + (kMseMaxBlocks + 1) * 4) : tail;
  L.fb_slot_bytes = L.fb_layer_bytes * d.n_layers;
  long w = 0;
  if (d.block == ADAPTRA_BLOCK_GPT) {
    long PT = L.flash ? 0 : (long)d.b * d.n_heads * d.T * d.T;
    L.w_S = 0;
    L.w_dS = align256(PT * 4);
    L.w_do = align256(L.w_dS + PT * e);
    L.w_D = align256(L.w_do + R * D * e);
    L.w_dq = align256(L.w_D + (long)d.b * d.n_heads * d.T * 4);
    w = L.flash ? align256(L.w_dq + R * D * 4) : L.w_dq;
  }
  // deterministic column-sum workspace (bias / LN parameter gradients of W):
  // partials [2][ceil(R/256)][N] fp32 and one ticket per 64-column strip for
  // every sum of a two-slot W (the grouped launch runs them all at once);
  // per layer the sums cover 7 d + d_ff columns (GPT; MLP: d + d_ff)
  const long cols = 2L * d.n_layers * (7 * D + F);
  L.cs_floats = 2 * ((R + 255) / 256) * cols;
  L.cs_tickets = cols / 64 + 2L * d.n_layers * 6 + 64;
  L.w_cs = align256(w);
  L.w_cnt = align256(L.w_cs + L.cs_floats * 4);
  w = align256(L.w_cnt + L.cs_tickets * 4);
  L.work_bytes = w;
  return ADAPTRA_OK;
}

// Parameter offsets (elements) of layer l inside wts / vecs.
struct ParamOff {
  long Wqkv, Wo, W1, W2;                       // wts
  long ln1_g, ln1_b, bqkv, bo, ln2_g, ln2_b, b1, b2;  // vecs
};
static long wts_per_layer(const adaptra_stage_desc_t& d) {
  long D = d.d, F = d.d_ff;
  return d.block == ADAPTRA_BLOCK_GPT ? 3 * D * D + D * D + F * D + D * F : F * D + D * F;
}
static long vecs_per_layer(const adaptra_stage_desc_t& d) {
  long D = d.d, F = d.d_ff;
  return d.block == ADAPTRA_BLOCK_GPT ? 2 * D + 3 * D + D + 2 * D + F + D : F + D;
}
static ParamOff param_off(const adaptra_stage_desc_t& d, int l) {
  ParamOff p{};
  long D = d.d, F = d.d_ff;
  long w0 = wts_per_layer(d) * l, v0 = vecs_per_layer(d) * l;
  if (d.block == ADAPTRA_BLOCK_GPT) {
    p.Wqkv = w0;
    p.Wo = p.Wqkv + 3 * D * D;
    p.W1 = p.Wo + D * D;
    p.W2 = p.W1 + F * D;
    p.ln1_g = v0;
    p.ln1_b = p.ln1_g + D;
    p.bqkv = p.ln1_b + D;
    p.bo = p.bqkv + 3 * D;
    p.ln2_g = p.bo + D;
    p.ln2_b = p.ln2_g + D;
    p.b1 = p.ln2_b + D;
    p.b2 = p.b1 + F;
  } else {
    p.W1 = w0;
    p.W2 = p.W1 + F * D;
    p.b1 = v0;
    p.b2 = p.b1 + F;
  }
  return p;
}

template <typename T>
struct StageOps {
  adaptra_stage* s;
  cudaStream_t st;
  const adaptra_stage_desc_t& d() const { return s->d; }
  char* slot_base(int slot) const { return (char*)s->d.stash + (long)slot * s->L.slot_bytes; }
  char* lay(int slot, int l) const { return slot_base(slot) + (long)l * s->L.layer_bytes; }
  T* buf(int slot, int l, long off) const { return (T*)(lay(slot, l) + off); }
  T* fbb(int slot, int l, long off) const {
    return (T*)((char*)s->d.stash_fb + (long)s->fb_of[slot] * s->L.fb_slot_bytes + (long)l * s->L.fb_layer_bytes + off);
  }
  float* fbuf(int slot, int l, long off) const { return (float*)(lay(slot, l) + off); }
  const T* W(long off) const { return (const T*)s->d.wts + off; }
  const float* V(long off) const { return s->d.vecs + off; }
  float* GW(long off) const { return s->d.gwts + off; }
  float* GV(long off) const { return s->d.gvecs + off; }
  int dt() const { return s->d.dtype; }

  // layer input / output pointers
  const T* layer_in(int slot, int l) const {
    return l == 0 ? (const T*)s->x_in[slot] : (const T*)buf(slot, l, s->L.xl);
  }
  T* layer_out(int slot, int l, void* y_out) const {
    if (l + 1 < s->d.n_layers) return buf(slot, l + 1, s->L.xl);
    if (s->d.is_last) return (T*)(slot_base(slot) + s->L.yL);
    return (T*)y_out;
  }
  // gradient of layer l output
  const T* layer_dy(int slot, int l) const {
    if (l + 1 < s->d.n_layers) return buf(slot, l, s->L.dyl);
    return (const T*)s->dy_in[slot];
  }
  T* layer_dx(int slot, int l, void* dx_out) const {
    if (l > 0) return buf(slot, l - 1, s->L.dyl);
    return (T*)dx_out;  // may be null on the first stage
  }

  int F(int slot, void* y_out, const float* target, float* loss_acc) {
    const auto& D = d();
    const long R = s->R, Dm = D.d, Ff = D.d_ff;
    for (int l = 0; l < D.n_layers; ++l) {
      ParamOff p = param_off(D, l);
      const T* x = layer_in(slot, l);
      T* y = layer_out(slot, l, y_out);
      if (!y) return set_error(ADAPTRA_EINVAL, "stage_F: y_out is null on a non-last stage");
      if (D.block == ADAPTRA_BLOCK_MLP) {
        T* a = fbb(slot, l, s->L.a);
        T* g = buf(slot, l, s->L.g);
        TRY(GB(dt()).shape(R, Ff, Dm).A(x, Dm, R, Dm).B(W(p.W1), Dm, Ff, Dm).C(g, Ff).aux(a, Ff)
                .epi(ADAPTRA_EPI_GELU).bias(V(p.b1)).run(st));
        TRY(GB(dt()).shape(R, Dm, Ff).A(g, Ff, R, Ff).B(W(p.W2), Ff, Dm, Ff).C(y, Dm)
                .epi(ADAPTRA_EPI_RESID).bias(V(p.b2)).res(x, Dm).run(st));
        continue;
      }
      const int H = D.n_heads, Tn = D.T, b = D.b;
      const long dh = Dm / H;
      T* h1 = buf(slot, l, s->L.h1);
      T* qkv = fbb(slot, l, s->L.qkv);
      T* P = fbb(slot, l, s->L.P);
      T* o = buf(slot, l, s->L.o);
      T* y1 = buf(slot, l, s->L.y1);
      T* h2 = buf(slot, l, s->L.h2);
      T* a = fbb(slot, l, s->L.a);
      T* g = buf(slot, l, s->L.g);
      float* S = (float*)((char*)D.work + s->L.w_S);
      TRY(ln_fwd<T>(x, V(p.ln1_g), V(p.ln1_b), h1, fbuf(slot, l, s->L.mean1), fbuf(slot, l, s->L.rstd1), R, Dm, st));
      TRY(GB(dt()).shape(R, 3 * Dm, Dm).A(h1, Dm, R, Dm).B(W(p.Wqkv), Dm, 3 * Dm, Dm).C(qkv, 3 * Dm)
              .epi(ADAPTRA_EPI_STORE).bias(V(p.bqkv)).run(st));
      if (s->L.flash) {
        // fused causal attention: o and the per-row LSE (kept for B)
        TRY(attn_fwd_tc((const bf16*)qkv, (bf16*)o, (float*)P, b, H, Tn, (int)Dm, st));
      } else {
      // scores S[z] = q_h k_h^T / sqrt(dh), z = (sequence, head); causal tiles only
      const float scale = 1.f / std::sqrt((float)dh);
      TRY(GB(dt()).shape(Tn, Tn, dh).batch(b * H, H)
              .A(qkv, 3 * Dm, R, Dm, 0, Tn, 0, 0, dh)
              .B(qkv + Dm, 3 * Dm, R, Dm, 0, Tn, 0, 0, dh)
              .C(S, Tn, (long)H * Tn * Tn, (long)Tn * Tn).epi(ADAPTRA_EPI_STORE_F32, scale)
              .causal(ADAPTRA_CAUSAL_TILE).run(st));
      TRY(softmax_causal<T>(S, P, b * H, Tn, st));
      // o_h = P_h v_h  (B = v MN-major), only keys j <= query tile end
      TRY(GB(dt()).shape(Tn, dh, Tn).batch(b * H, H)
              .A(P, Tn, (long)b * H * Tn, Tn, 0, (long)H * Tn, Tn, 0, 0)
              .B(qkv + 2 * Dm, 3 * Dm, R, Dm, 1, Tn, 0, 0, dh)
              .C(o, Dm, (long)Tn * Dm, dh).causal(ADAPTRA_CAUSAL_KEND).run(st));
      }
      TRY(GB(dt()).shape(R, Dm, Dm).A(o, Dm, R, Dm).B(W(p.Wo), Dm, Dm, Dm).C(y1, Dm)
              .epi(ADAPTRA_EPI_RESID).bias(V(p.bo)).res(x, Dm).run(st));
      TRY(ln_fwd<T>(y1, V(p.ln2_g), V(p.ln2_b), h2, fbuf(slot, l, s->L.mean2), fbuf(slot, l, s->L.rstd2), R, Dm, st));
      TRY(GB(dt()).shape(R, Ff, Dm).A(h2, Dm, R, Dm).B(W(p.W1), Dm, Ff, Dm).C(g, Ff).aux(a, Ff)
              .epi(ADAPTRA_EPI_GELU).bias(V(p.b1)).run(st));
      TRY(GB(dt()).shape(R, Dm, Ff).A(g, Ff, R, Ff).B(W(p.W2), Ff, Dm, Ff).C(y, Dm)
              .epi(ADAPTRA_EPI_RESID).bias(V(p.b2)).res(y1, Dm).run(st));
    }
    if (D.is_last) {
      if (!target || !loss_acc) return set_error(ADAPTRA_EINVAL, "stage_F: last stage needs target and loss_acc");
      const T* y = (const T*)(slot_base(slot) + s->L.yL);
      T* seed = (T*)(slot_base(slot) + s->L.seed);
      TRY(mse_loss<T>(y, target, seed, loss_acc, (float*)(slot_base(slot) + s->L.lpart), s->R * D.d,
                      D.n_microbatches, st));
      s->dy_in[slot] = seed;
    }
    return ADAPTRA_OK;
  }

  int B(int slot, void* dx_out) {
    const auto& D = d();
    const long R = s->R, Dm = D.d, Ff = D.d_ff;
    for (int l = D.n_layers - 1; l >= 0; --l) {
      ParamOff p = param_off(D, l);
      const T* dy = layer_dy(slot, l);
      T* dx = layer_dx(slot, l, dx_out);
      const T* x = layer_in(slot, l);
      T* a = fbb(slot, l, s->L.a);
      T* da = buf(slot, l, s->L.da);
      // da = (dy W2) * gelu'(a)     (W2 [d, dff] read MN-major)
      TRY(GB(dt()).shape(R, Ff, Dm).A(dy, Dm, R, Dm).B(W(p.W2), Ff, Dm, Ff, 1).C(da, Ff)
              .epi(ADAPTRA_EPI_DGELU).aux(a, Ff).run(st));
      if (D.block == ADAPTRA_BLOCK_MLP) {
        if (dx)  // dx = dy + da W1
          TRY(GB(dt()).shape(R, Dm, Ff).A(da, Ff, R, Ff).B(W(p.W1), Dm, Ff, Dm, 1).C(dx, Dm)
                  .epi(ADAPTRA_EPI_RESID).res(dy, Dm).run(st));
        continue;
      }
      const int H = D.n_heads, Tn = D.T, b = D.b;
      const long dh = Dm / H;
      T* qkv = fbb(slot, l, s->L.qkv);
      T* P = fbb(slot, l, s->L.P);
      T* o = buf(slot, l, s->L.o);
      T* y1 = buf(slot, l, s->L.y1);
      T* dqkv = buf(slot, l, s->L.dqkv);
      T* dy1 = buf(slot, l, s->L.dy1);
      T* dh2 = buf(slot, l, s->L.dh2);
      T* dh1 = buf(slot, l, s->L.dh1);
      T* dS = (T*)((char*)D.work + s->L.w_dS);
      T* dO = (T*)((char*)D.work + s->L.w_do);
      float* Dv = (float*)((char*)D.work + s->L.w_D);
      // dh2 = da W1 ; dy1 = dy + LN2_bwd(dh2)
      TRY(GB(dt()).shape(R, Dm, Ff).A(da, Ff, R, Ff).B(W(p.W1), Dm, Ff, Dm, 1).C(dh2, Dm).run(st));
      TRY(ln_bwd<T>(dh2, y1, fbuf(slot, l, s->L.mean2), fbuf(slot, l, s->L.rstd2), V(p.ln2_g), dy, dy1, R, Dm, st));
      // do = dy1 Wo ; D = rowsum(do o o) per head (fused into the GEMM's epilogue on the tcgen05 path)
      if (s->L.flash && Dm % 256 == 0 && Dm >= 2048) {
        TRY(GB(dt()).shape(R, Dm, Dm).A(dy1, Dm, R, Dm).B(W(p.Wo), Dm, Dm, Dm, 1).C(dO, Dm)
                .epi(ADAPTRA_EPI_STORE_ROWDOT).aux(o, Dm).rowv(Dv, Tn, H).run(st));
      } else {
        TRY(GB(dt()).shape(R, Dm, Dm).A(dy1, Dm, R, Dm).B(W(p.Wo), Dm, Dm, Dm, 1).C(dO, Dm).run(st));
        TRY(attn_rowdot<T>(dO, o, Dv, b, H, Tn, dh, Dm, st));
      }
      if (s->L.flash) {
        float* dq_acc = (float*)((char*)D.work + s->L.w_dq);
        TRY(attn_bwd_tc((const bf16*)qkv, (const bf16*)dO, (const float*)P, Dv, (bf16*)dqkv, dq_acc, b, H, Tn, (int)Dm,
                        st));
      } else {
      const float scale = 1.f / std::sqrt((float)dh);
      // dS = P * (do_h v_h^T - D) / sqrt(dh)
      TRY(GB(dt()).shape(Tn, Tn, dh).batch(b * H, H)
              .A(dO, Dm, R, Dm, 0, Tn, 0, 0, dh)
              .B(qkv + 2 * Dm, 3 * Dm, R, Dm, 0, Tn, 0, 0, dh)
              .C(dS, Tn, (long)H * Tn * Tn, (long)Tn * Tn)
              .aux(P, Tn, (long)H * Tn * Tn, (long)Tn * Tn).rowv(Dv, (long)H * Tn, Tn)
              .epi(ADAPTRA_EPI_DSOFTMAX, scale).causal(ADAPTRA_CAUSAL_TILE).run(st));
      // dq = dS k   (k read MN-major)
      TRY(GB(dt()).shape(Tn, dh, Tn).batch(b * H, H)
              .A(dS, Tn, (long)b * H * Tn, Tn, 0, (long)H * Tn, Tn, 0, 0)
              .B(qkv + Dm, 3 * Dm, R, Dm, 1, Tn, 0, 0, dh)
              .C(dqkv, 3 * Dm, (long)Tn * 3 * Dm, dh).causal(ADAPTRA_CAUSAL_KEND).run(st));
      // dk = dS^T q   (dS and q read MN-major)
      TRY(GB(dt()).shape(Tn, dh, Tn).batch(b * H, H)
              .A(dS, Tn, (long)b * H * Tn, Tn, 1, (long)H * Tn, Tn, 0, 0)
              .B(qkv, 3 * Dm, R, Dm, 1, Tn, 0, 0, dh)
              .C(dqkv + Dm, 3 * Dm, (long)Tn * 3 * Dm, dh).causal(ADAPTRA_CAUSAL_KSTART).run(st));
      // dv = P^T do
      TRY(GB(dt()).shape(Tn, dh, Tn).batch(b * H, H)
              .A(P, Tn, (long)b * H * Tn, Tn, 1, (long)H * Tn, Tn, 0, 0)
              .B(dO, Dm, R, Dm, 1, Tn, 0, 0, dh)
              .C(dqkv + 2 * Dm, 3 * Dm, (long)Tn * 3 * Dm, dh).causal(ADAPTRA_CAUSAL_KSTART).run(st));
      }
      // dh1 = dqkv Wqkv ; dx = dy1 + LN1_bwd(dh1)
      TRY(GB(dt()).shape(R, Dm, 3 * Dm).A(dqkv, 3 * Dm, R, 3 * Dm).B(W(p.Wqkv), Dm, 3 * Dm, Dm, 1).C(dh1, Dm)
              .run(st));
      if (dx)
        TRY(ln_bwd<T>(dh1, x, fbuf(slot, l, s->L.mean1), fbuf(slot, l, s->L.rstd1), V(p.ln1_g), dy1, dx, R, Dm, st));
    }
    return ADAPTRA_OK;
  }

  // W of 1..4 slots (consecutive W ops of the stage's order) as one launch
  // whose products run over K = n b T: the fp32 gradient is read-modified-
  // written once per group instead of once per microbatch, and every tile's
  // epilogue is amortised over n times the K loop
  int Wop(const int* slots, int n) {
    std::vector<adaptra_gemm_desc_t> dw[4];
    std::vector<float*> db[4];     // per product: its bias gradient (A = dY of the product)
    std::vector<ColsumJob> cs[4];  // per slot: the slots' sums add into the same gradients
    for (int k = 0; k < n; ++k) collect_w(slots[k], dw[k], cs[k], db[k]);
    // bias gradients summed inside the grouped dW launch from its staged dY
    // tiles ($ADAPTRA_DB_FUSED=0: separate column-sum launches, as before)
    static const bool db_fused = !(getenv("ADAPTRA_DB_FUSED") && atoi(getenv("ADAPTRA_DB_FUSED")) == 0);
    std::vector<float*> fused_db;
    if (dt() == ADAPTRA_BF16) {
      for (size_t i = 0; i < dw[0].size(); i += 24) {
        const adaptra_gemm_desc_t* more[3];
        for (int k = 1; k < n; ++k) more[k - 1] = dw[k].data() + i;
        const int m = (int)std::min<size_t>(24, dw[0].size() - i);
        bool fused = false;
        TRY(gemm_tc_grouped(dw[0].data() + i, m, st, more, n - 1, db_fused ? db[0].data() + i : nullptr, &fused));
        if (fused) fused_db.insert(fused_db.end(), db[0].begin() + i, db[0].begin() + i + m);
      }
    } else {
      for (int k = 0; k < n; ++k)
        for (auto& g : dw[k]) TRY(gemm_simt(g, st));
    }
    // Column sums (bias gradients not fused above, LN parameter gradients):
    // one deterministic launch per sum by default.  All of the op's sums in
    // one grouped launch (ADAPTRA_COLSUM_GROUPED=1) take 9 % off a 3-layer C1
    // W op run alone (profiles/r02_op_bench_pp.jsonl), but with 8 stages
    // sharing the GPU the step is 3.8 % slower (3 + 3 alternating runs,
    // r02_colsum_step_ab.txt): its ~1.5k-block grid crowds the other stages.
    static const bool cs_grouped = getenv("ADAPTRA_COLSUM_GROUPED") && atoi(getenv("ADAPTRA_COLSUM_GROUPED")) == 1;
    const long R = s->R;
    float* part = (float*)((char*)s->d.work + s->L.w_cs);
    unsigned* cnt = (unsigned*)((char*)s->d.work + s->L.w_cnt);
    for (int k = 0; k < n; ++k) {
      std::vector<ColsumJob> jobs;
      for (const auto& j : cs[k])
        if (j.ln || std::find(fused_db.begin(), fused_db.end(), j.out_a) == fused_db.end()) jobs.push_back(j);
      if (cs_grouped) {
        // one launch per slot: a launch's jobs must not share an output (the
        // last block of a strip adds into it without atomics)
        if (!jobs.empty())
          TRY(colsum_grouped<T>(jobs.data(), (int)jobs.size(), (int)R, st, part, cnt, s->L.cs_floats,
                                s->L.cs_tickets));
        continue;
      }
      for (const auto& j : jobs) {
        if (j.ln)
          TRY(ln_param_grad<T>((const T*)j.y, (const T*)j.x, j.mean, j.rstd, j.out_a, j.out_b, (int)R, j.N, st, part,
                               cnt));
        else
          TRY(col_sum<T>((const T*)j.y, j.out_a, (int)R, j.N, st, part, cnt));
      }
    }
    return ADAPTRA_OK;
  }

  void collect_w(int slot, std::vector<adaptra_gemm_desc_t>& dw, std::vector<ColsumJob>& cs, std::vector<float*>& db) {
    const auto& D = d();
    const long R = s->R, Dm = D.d, Ff = D.d_ff;
    // every dW += X^T dY product of the op is independent: collect them and run
    // them as grouped persistent launches (bias / LN parameter sums after)
    dw.reserve(4 * D.n_layers);
    cs.reserve(cs.size() + 6 * D.n_layers);
    for (int l = D.n_layers - 1; l >= 0; --l) {
      ParamOff p = param_off(D, l);
      const T* dy = layer_dy(slot, l);
      const T* x = layer_in(slot, l);
      T* g = buf(slot, l, s->L.g);
      T* da = buf(slot, l, s->L.da);
      // dW2 += dy^T g ; db2 += sum dy
      dw.push_back(GB(dt()).shape(Dm, Ff, R).A(dy, Dm, R, Dm, 1).B(g, Ff, R, Ff, 1).C(GW(p.W2), Ff)
              .epi(ADAPTRA_EPI_ACC_F32).g);
      db.push_back(GV(p.b2));
      cs.push_back(ColsumJob{dy, nullptr, nullptr, nullptr, GV(p.b2), nullptr, (int)(Dm), 0, 0, 0});
      if (D.block == ADAPTRA_BLOCK_MLP) {
        dw.push_back(GB(dt()).shape(Ff, Dm, R).A(da, Ff, R, Ff, 1).B(x, Dm, R, Dm, 1).C(GW(p.W1), Dm)
                .epi(ADAPTRA_EPI_ACC_F32).g);
        db.push_back(GV(p.b1));
        cs.push_back(ColsumJob{da, nullptr, nullptr, nullptr, GV(p.b1), nullptr, (int)(Ff), 0, 0, 0});
        continue;
      }
      T* h1 = buf(slot, l, s->L.h1);
      T* o = buf(slot, l, s->L.o);
      T* y1 = buf(slot, l, s->L.y1);
      T* h2 = buf(slot, l, s->L.h2);
      T* dqkv = buf(slot, l, s->L.dqkv);
      T* dy1 = buf(slot, l, s->L.dy1);
      T* dh2 = buf(slot, l, s->L.dh2);
      T* dh1 = buf(slot, l, s->L.dh1);
      dw.push_back(GB(dt()).shape(Ff, Dm, R).A(da, Ff, R, Ff, 1).B(h2, Dm, R, Dm, 1).C(GW(p.W1), Dm)
              .epi(ADAPTRA_EPI_ACC_F32).g);
      db.push_back(GV(p.b1));
      cs.push_back(ColsumJob{da, nullptr, nullptr, nullptr, GV(p.b1), nullptr, (int)(Ff), 0, 0, 0});
      cs.push_back(ColsumJob{dh2, y1, fbuf(slot, l, s->L.mean2), fbuf(slot, l, s->L.rstd2), GV(p.ln2_g), GV(p.ln2_b), (int)Dm, 1, 0, 0});
      dw.push_back(GB(dt()).shape(Dm, Dm, R).A(dy1, Dm, R, Dm, 1).B(o, Dm, R, Dm, 1).C(GW(p.Wo), Dm)
              .epi(ADAPTRA_EPI_ACC_F32).g);
      db.push_back(GV(p.bo));
      cs.push_back(ColsumJob{dy1, nullptr, nullptr, nullptr, GV(p.bo), nullptr, (int)(Dm), 0, 0, 0});
      dw.push_back(GB(dt()).shape(3 * Dm, Dm, R).A(dqkv, 3 * Dm, R, 3 * Dm, 1).B(h1, Dm, R, Dm, 1).C(GW(p.Wqkv), Dm)
              .epi(ADAPTRA_EPI_ACC_F32).g);
      db.push_back(GV(p.bqkv));
      cs.push_back(ColsumJob{dqkv, nullptr, nullptr, nullptr, GV(p.bqkv), nullptr, (int)(3 * Dm), 0, 0, 0});
      cs.push_back(ColsumJob{dh1, x, fbuf(slot, l, s->L.mean1), fbuf(slot, l, s->L.rstd1), GV(p.ln1_g), GV(p.ln1_b), (int)Dm, 1, 0, 0});
    }
    // drop empty products (and their bias entries, kept parallel)
    size_t w = 0;
    for (size_t i = 0; i < dw.size(); ++i)
      if (dw[i].M != 0 && dw[i].N != 0) {
        dw[w] = dw[i];
        db[w++] = db[i];
      }
    dw.resize(w);
    db.resize(w);
  }
};

}  // namespace adaptra

using namespace adaptra;

namespace adaptra {
int stage_n_slots(adaptra_stage_t s) { return s->d.n_slots; }
int stage_device(adaptra_stage_t s) { return s->dev; }
// N4 stash offload (exec.cpp): a slot's bytes and its host-side metadata
// (the layer-0 input and top-layer gradient pointers W reads) move together.
void* stage_slot_base(adaptra_stage_t s, int slot) { return (char*)s->d.stash + (long)slot * s->L.slot_bytes; }
int64_t stage_slot_nbytes(adaptra_stage_t s) { return s->L.slot_bytes; }
void stage_get_meta(adaptra_stage_t s, int slot, const void** x_in, const void** dy_in) {
  *x_in = s->x_in[slot];
  *dy_in = s->dy_in[slot];
}
// Restore metadata saved from slot `from` into slot `to`: pointers that
// pointed inside slot `from` (the last stage's MSE seed) are rebased.
void stage_set_meta(adaptra_stage_t s, int to, int from, const void* x_in, const void* dy_in) {
  const char* b0 = (const char*)stage_slot_base(s, from);
  const char* b1 = (const char*)stage_slot_base(s, to);
  auto rebase = [&](const void* p) -> const void* {
    const char* c = (const char*)p;
    return (c >= b0 && c < b0 + s->L.slot_bytes) ? b1 + (c - b0) : p;
  };
  s->x_in[to] = rebase(x_in);
  s->dy_in[to] = rebase(dy_in);
}
}  // namespace adaptra

extern "C" int64_t adaptra_stage_slot_bytes(const adaptra_stage_desc_t* d) {
  SlotLayout L;
  if (!d || compute_layout(*d, L)) return -1;
  return L.slot_bytes;
}
extern "C" int64_t adaptra_stage_slot_fb_bytes(const adaptra_stage_desc_t* d) {
  SlotLayout L;
  if (!d || compute_layout(*d, L)) return -1;
  return L.fb_slot_bytes;
}
extern "C" int64_t adaptra_stage_work_bytes(const adaptra_stage_desc_t* d) {
  SlotLayout L;
  if (!d || compute_layout(*d, L)) return -1;
  return L.work_bytes;
}
extern "C" int64_t adaptra_stage_wts_elems(const adaptra_stage_desc_t* d) {
  return d ? wts_per_layer(*d) * d->n_layers : -1;
}
extern "C" int64_t adaptra_stage_vecs_elems(const adaptra_stage_desc_t* d) {
  return d ? vecs_per_layer(*d) * d->n_layers : -1;
}

extern "C" int adaptra_stage_create(const adaptra_stage_desc_t* d, adaptra_stage_t* out) {
  if (!d || !out) return set_error(ADAPTRA_EINVAL, "stage_create: null");
  auto* s = new adaptra_stage();
  s->d = *d;
  int rc = compute_layout(*d, s->L);
  if (rc) {
    delete s;
    return rc;
  }
  if (!d->wts || !d->vecs || !d->gwts || !d->gvecs || !d->stash || d->n_slots < 1 || !d->stash_fb ||
      d->n_slots_fb < 1 ||
      !d->work) {
    delete s;
    return set_error(ADAPTRA_EINVAL, "stage_create: missing buffers");
  }
  s->R = (long)d->b * d->T;
  cudaPointerAttributes pa;
  if (cudaPointerGetAttributes(&pa, d->wts) == cudaSuccess && pa.type == cudaMemoryTypeDevice) s->dev = pa.device;
  else cudaGetDevice(&s->dev);
  s->x_in.assign(d->n_slots, nullptr);
  s->dy_in.assign(d->n_slots, nullptr);
  if (s->L.flash && s->L.work_bytes > 0) {
    // the fused attention backward accumulates dQ with TMA reduce-add; the
    // finalize kernel re-zeroes it after every use
    cudaMemset((char*)d->work + s->L.w_dq, 0, (size_t)s->R * d->d * 4);
  }
  // column-sum tickets start at 0 (the last block of a strip resets its own)
  cudaMemset((char*)d->work + s->L.w_cnt, 0, (size_t)(s->L.work_bytes - s->L.w_cnt));
  cudaDeviceSynchronize();
  s->fb_of.assign(d->n_slots, -1);
  for (int k = d->n_slots_fb - 1; k >= 0; --k) s->fb_free.push_back(k);
  *out = s;
  return ADAPTRA_OK;
}

extern "C" int adaptra_stage_destroy(adaptra_stage_t s) {
  delete s;
  return ADAPTRA_OK;
}

extern "C" int adaptra_stage_F(adaptra_stage_t s, int32_t slot, const void* x_in, void* y_out, const float* target,
                               float* loss_acc, void* stream) {
  if (!s || slot < 0 || slot >= s->d.n_slots || !x_in) return set_error(ADAPTRA_EINVAL, "stage_F: bad args");
  if (s->fb_of[slot] >= 0) return set_error(ADAPTRA_EINVAL, "stage_F: slot still holds an un-consumed F");
  if (s->fb_free.empty()) return set_error(ADAPTRA_ENOMEM, "stage_F: F->B stash pool exhausted");
  s->fb_of[slot] = s->fb_free.back();
  s->fb_free.pop_back();
  s->x_in[slot] = x_in;
  s->dy_in[slot] = nullptr;
  if (s->d.dtype == ADAPTRA_BF16) return StageOps<bf16>{s, (cudaStream_t)stream}.F(slot, y_out, target, loss_acc);
  return StageOps<float>{s, (cudaStream_t)stream}.F(slot, y_out, target, loss_acc);
}

extern "C" int adaptra_stage_B(adaptra_stage_t s, int32_t slot, const void* dy_in, void* dx_out, void* stream) {
  if (!s || slot < 0 || slot >= s->d.n_slots) return set_error(ADAPTRA_EINVAL, "stage_B: bad args");
  if (!s->d.is_last) {
    if (!dy_in) return set_error(ADAPTRA_EINVAL, "stage_B: dy_in required on a non-last stage");
    s->dy_in[slot] = dy_in;
  } else if (!s->dy_in[slot]) {
    return set_error(ADAPTRA_EINVAL, "stage_B: F was not run for this slot");
  }
  if (!s->d.is_first && !dx_out) return set_error(ADAPTRA_EINVAL, "stage_B: dx_out required on a non-first stage");
  if (s->fb_of[slot] < 0) return set_error(ADAPTRA_EINVAL, "stage_B: no F for this slot");
  int rc = s->d.dtype == ADAPTRA_BF16
               ? StageOps<bf16>{s, (cudaStream_t)stream}.B(slot, s->d.is_first ? nullptr : dx_out)
               : StageOps<float>{s, (cudaStream_t)stream}.B(slot, s->d.is_first ? nullptr : dx_out);
  // the F->B buffers are free once B's kernels are enqueued (stream order)
  s->fb_free.push_back(s->fb_of[slot]);
  s->fb_of[slot] = -1;
  return rc;
}

extern "C" int adaptra_stage_W(adaptra_stage_t s, int32_t slot, void* stream) {
  if (!s || slot < 0 || slot >= s->d.n_slots || !s->dy_in[slot]) return set_error(ADAPTRA_EINVAL, "stage_W: bad args");
  if (s->d.dtype == ADAPTRA_BF16) return StageOps<bf16>{s, (cudaStream_t)stream}.Wop(&slot, 1);
  return StageOps<float>{s, (cudaStream_t)stream}.Wop(&slot, 1);
}

extern "C" int adaptra_stage_Wn(adaptra_stage_t s, const int32_t* slots, int32_t n, void* stream) {
  if (!s || !slots || n < 1 || n > 4) return set_error(ADAPTRA_EINVAL, "stage_Wn: 1..4 slots");
  for (int k = 0; k < n; ++k) {
    if (slots[k] < 0 || slots[k] >= s->d.n_slots || !s->dy_in[slots[k]]) return set_error(ADAPTRA_EINVAL, "stage_Wn: bad slot");
    for (int m = 0; m < k; ++m)
      if (slots[m] == slots[k]) return set_error(ADAPTRA_EINVAL, "stage_Wn: repeated slot");
  }
  const int sl[4] = {slots[0], n > 1 ? slots[1] : 0, n > 2 ? slots[2] : 0, n > 3 ? slots[3] : 0};
  if (s->d.dtype == ADAPTRA_BF16) return StageOps<bf16>{s, (cudaStream_t)stream}.Wop(sl, n);
  return StageOps<float>{s, (cudaStream_t)stream}.Wop(sl, n);
}

extern "C" int adaptra_stage_W2(adaptra_stage_t s, int32_t slot_a, int32_t slot_b, void* stream) {
  const int32_t sl[2] = {slot_a, slot_b};
  return adaptra_stage_Wn(s, sl, 2, stream);
}

extern "C" int adaptra_stage_zero_grads(adaptra_stage_t s, void* stream) {
  if (!s) return set_error(ADAPTRA_EINVAL, "zero_grads: null");
  cudaStream_t st = (cudaStream_t)stream;
  ADAPTRA_CUDA_TRY(cudaMemsetAsync(s->d.gwts, 0, adaptra_stage_wts_elems(&s->d) * 4, st));
  ADAPTRA_CUDA_TRY(cudaMemsetAsync(s->d.gvecs, 0, adaptra_stage_vecs_elems(&s->d) * 4, st));
  return ADAPTRA_OK;
}
