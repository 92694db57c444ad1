/*
 * adaptra.h -- C-ABI of libadaptra.so, the B200-native hot path of Adaptra
 * (arXiv 2504.19232): the zero-bubble (ZB) pipeline-parallel training step.
 *
 * Citations: P:<line> = PAPER.md (main.tex copy); R<k> = reading k in
 * DESIGN.md §3 (where the paper is silent or ambiguous).
 *
 * Conventions (all entry points)
 *  - Every call returns int32 status: ADAPTRA_OK (0) or a negative ADAPTRA_E*
 *    code; adaptra_last_error() returns a thread-local message for the last
 *    failure on the calling thread.  No C++ exception crosses the ABI.
 *  - Time is int64 "ticks" (the runtime uses nanoseconds).  Planner and
 *    schedule inputs are exact integers: results are bit-identical to the CPU
 *    oracle on the same inputs.
 *  - Memory ownership: the caller allocates every output array (host arrays
 *    for planning calls; device buffers for stage calls).  Weights, gradients,
 *    stash arenas and workspaces are caller-owned (the Python binding
 *    allocates them with torch); the library only borrows raw pointers.
 *    Library-allocated: opaque handles (stage, inbox, outbox, exec) and the
 *    inbox mailboxes/flags/host rings (whole cudaMalloc / shm allocations so
 *    they can be exported across processes); all are freed by the matching
 *    *_destroy / *_close call.
 *  - Device work is enqueued on caller-supplied cudaStream_t (passed as void*).
 *    Asynchronous CUDA faults surface as ADAPTRA_ECUDA from a later call.
 *  - Planning calls are pure and reentrant.  A stage or link handle must be
 *    driven by one host thread at a time.
 */
#ifndef ADAPTRA_H
#define ADAPTRA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status */
#define ADAPTRA_OK 0
#define ADAPTRA_EINVAL (-1)    /* bad argument                                  */
#define ADAPTRA_EPLAN (-2)     /* warm-up plan violates the Lemma, x_0 > N or x_{S-1} < 1 */
#define ADAPTRA_EDEADLOCK (-3) /* replay of a fixed order cannot progress       */
#define ADAPTRA_ECUDA (-4)     /* CUDA runtime/driver error                      */
#define ADAPTRA_ENOMEM (-5)    /* output capacity too small / allocation failed  */
#define ADAPTRA_ELINK (-6)     /* transport error                                */
#define ADAPTRA_ETOOBIG (-7)   /* problem exceeds a kernel limit                 */

const char* adaptra_last_error(void);

/* Library build/version string (also proves the .so loaded). */
const char* adaptra_version(void);

/* ================================================================ planning
 * Pure host integer code (csrc/sched/).  Bit-exact with oracle/sched.py.
 */

/* Operator kinds: forward, backward-input, backward-weight. */
#define ADAPTRA_OP_F 0
#define ADAPTRA_OP_B 1
#define ADAPTRA_OP_W 2

/* One scheduled operator.  mb is 1-based (the paper's F_1..F_N). */
typedef struct adaptra_op {
  int32_t kind;  /* ADAPTRA_OP_* */
  int32_t mb;    /* microbatch, 1..N */
  int64_t start; /* ticks */
  int64_t end;   /* ticks */
} adaptra_op_t;

/* adaptra_schedule / adaptra_replay flags */
#define ADAPTRA_SEL_PAPER 0u /* literal greedy SelectOp (R7, default)                 */
#define ADAPTRA_SEL_CAP 1u   /* F eligible only while (#F - #B) < x_i (1F1B / ZB-H1)   */
#define ADAPTRA_MERGE_W 2u   /* 1F1B: W folded into B, no W ops (R10)                  */

/* Alg. 1 GetInitWarmupFwds: x_max = min(floor(M/M^F), N) (R12),
 * x_0 = x_max, balanced slackness.  x_out[S].  EINVAL if S < 2 or x_max < 1. */
int adaptra_plan_init(int32_t S, int32_t N, int64_t mem_capacity, int64_t mem_per_act, int32_t* x_out);

/* Alg. 2 GetAdaptedWarmupFwds with the R11 clamps:
 * Delta_i = max(0, min(N-2S, max(ceil((tF_i+tB_i+2c_i)/(tF_{i+1}+tB_{i+1})), 2))),
 * x_i = min(N, x_{i+1} + Delta_i), x_{S-1} = 1.  tF,tB[S], c[S-1] (finite, >= 0). */
int adaptra_plan_adapt(int32_t S, int32_t N, const int64_t* tF, const int64_t* tB, const int64_t* c,
                       int32_t* x_out);

/* Eq. 1 per link: ok_out[i] = tF_i + tB_i + 2c_i <= (x_i - x_{i+1})(tF_{i+1} + tB_{i+1}). */
int adaptra_eq1_holds(int32_t S, const int64_t* tF, const int64_t* tB, const int64_t* c, const int32_t* x,
                      uint8_t* ok_out);

/* Alg. 4 Schedule with Alg. 3 SelectOp, readings R1-R10:
 * discrete-time simulation with step delta >= 1 tick.  Writes stage i's ops in
 * execution order to ops_out[i*3N .. i*3N + n_ops_out[i]) (capacity S*3N).
 * x[S] must satisfy the Lemma, x_0 <= N, x_{S-1} >= 1 (else EPLAN).
 * makespan_out = max end (R9); steps_out = number of delta steps. */
int adaptra_schedule(int32_t S, int32_t N, const int64_t* tF, const int64_t* tB, const int64_t* tW,
                     const int64_t* c, const int32_t* x, int64_t delta, uint32_t flags, adaptra_op_t* ops_out,
                     int32_t* n_ops_out, int64_t* makespan_out, int64_t* steps_out);

/* Event-driven replay of a fixed per-stage order (start/end of `order` are
 * ignored) under latencies c: every op starts at max(stage free, deps ready)
 * with the dependency rules of P:1743-1753 (+R8).  timed_out has the layout of
 * ops_out above.  EDEADLOCK if no stage can progress. */
int adaptra_replay(int32_t S, int32_t N, const int64_t* tF, const int64_t* tB, const int64_t* tW,
                   const int64_t* c, const adaptra_op_t* order, const int32_t* n_ops, uint32_t flags,
                   adaptra_op_t* timed_out, int64_t* makespan_out);

/* One violation found by adaptra_validate / adaptra_validate_plan. */
typedef struct adaptra_violation {
  int32_t code;  /* ADAPTRA_V_*                                                  */
  int32_t stage; /* stage of the offending op (plan codes: the index i of x_i)   */
  int32_t kind;  /* ADAPTRA_OP_* of the offending op (-1 for plan codes)        */
  int32_t mb;    /* its microbatch, 1..N (0 for plan codes)                      */
} adaptra_violation_t;

#define ADAPTRA_V_BADOP 1    /* kind not F/B/W, mb outside 1..N, or a W op in a MERGE_W schedule (R10) */
#define ADAPTRA_V_DUP 2      /* the op appears twice on its stage                                      */
#define ADAPTRA_V_MISSING 3  /* one of the stage's 3N (2N with MERGE_W) ops is absent                  */
#define ADAPTRA_V_DURATION 4 /* end - start != the stage's op time (B + W with MERGE_W)                 */
#define ADAPTRA_V_OVERLAP 5  /* starts before the previous op of its stage ended (P:2754 busy())        */
#define ADAPTRA_V_DEP 6      /* starts before a dependency's end + link latency (R1, R2,
                                R8); one entry per violated dependency                                 */
#define ADAPTRA_V_NONMONO 7  /* plan: x_i < x_{i+1} (the Lemma); stage = i                 */
#define ADAPTRA_V_X_LAST 8   /* plan: x_{S-1} < 1 (Alg. 1/2 end at 1)                  */
#define ADAPTRA_V_X0_GT_N 9  /* plan: x_0 > N (R11)                                                     */

/* Check a timed schedule (layout of adaptra_schedule's ops_out) against the
 * problem's constraints (violations are values, not errors).
 * Writes the first min(cap, total) violations to violations_out (caller-owned,
 * may be NULL when cap == 0) in stage order and sets *n_violations_out to the
 * total (0 = valid).  EINVAL on bad pointers or n_ops outside 0..3N. */
int adaptra_validate(int32_t S, int32_t N, const int64_t* tF, const int64_t* tB, const int64_t* tW,
                     const int64_t* c, const adaptra_op_t* ops, const int32_t* n_ops, uint32_t flags,
                     adaptra_violation_t* violations_out, int32_t cap, int32_t* n_violations_out);
/* Check a warm-up plan x[S] (codes ADAPTRA_V_NONMONO / X_LAST / X0_GT_N), same
 * output convention. */
int adaptra_validate_plan(int32_t S, int32_t N, const int32_t* x, adaptra_violation_t* violations_out, int32_t cap,
                          int32_t* n_violations_out);

/* 1F1B warm-up counts x_i = min(S - i, N) (R21 baseline).  x_out[S]. */
int adaptra_plan_1f1b(int32_t S, int32_t N, int32_t* x_out);
/* R26 (no host offload of the F->B stash): x_i <- min(x_i, cap_i), then the
 * Lemma restored from the last stage up, x_i <- max(x_i, x_{i+1}).  In place. */
int adaptra_clamp_plan(int32_t S, const int32_t* cap, int32_t* x_inout);
/* R10: delta = max(1, floor(t_o / ratio)), t_o = the largest op time (ratio 30).
 * Returns delta (1 on bad arguments). */
int64_t adaptra_default_delta(int32_t S, const int64_t* tF, const int64_t* tB, const int64_t* tW, int32_t ratio);

/* ---------------------------------------------------------------- planner
 * One schedule arm per object, so that the per-iteration planning decision of
 * the bench / training loop is one C call (DESIGN.md §3 R18, R21, R26):
 *  ADAPTRA_ARM_1F1B      x_i = min(S-i, N), Schedule(SEL_CAP | MERGE_W) at c = 0, frozen;
 *  ADAPTRA_ARM_ZB        x = Alg. 2 at c = 0, Schedule(SEL_PAPER) at c = 0, frozen (R21);
 *  ADAPTRA_ARM_ADAPTIVE  x_init = desc.x_init if given, else Alg. 1 (mem_capacity /
 *                        mem_per_act, R12) clamped to x_cap (R26) if mem_per_act > 0,
 *                        else Alg. 2 at c = 0.  At each step whose c differs from the
 *                        previous step's (R18): every link nominal (c = 0) -> x_init;
 *                        else if Eq. 1 fails on some link under the current x -> Alg. 2
 *                        with c, clamped to x_cap (R26); else x is kept.  The orders are
 *                        Schedule(SEL_PAPER, c, x, delta).  A profile passed with
 *                        adaptra_planner_set_profile is adopted at the next such re-plan.
 * delta = adaptra_default_delta(profile, ratio).  Everything is integer and
 * bit-exact with the oracle (oracle.sched.adaptive_orders). */
#define ADAPTRA_ARM_1F1B 0
#define ADAPTRA_ARM_ZB 1
#define ADAPTRA_ARM_ADAPTIVE 2
#define ADAPTRA_MAX_STAGES 64

typedef struct adaptra_planner_desc {
  int32_t S, N, arm, ratio;          /* ratio: ceil(t_o/delta) target, 0 = 30   */
  const int64_t *tF, *tB, *tW;       /* [S] op times in ticks (ns), each >= 1            */
  const int32_t* x_init;             /* [S] or NULL                                      */
  const int32_t* x_cap;              /* [S] device stash capacity per stage, or NULL      */
  int64_t mem_capacity, mem_per_act; /* Alg. 1 inputs M, M^F (used if mem_per_act > 0)   */
} adaptra_planner_desc_t;

typedef struct adaptra_plan_info {
  int64_t makespan, delta, replans;  /* the simulated T, the step, re-plans so far       */
  int64_t tF[ADAPTRA_MAX_STAGES], tB[ADAPTRA_MAX_STAGES], tW[ADAPTRA_MAX_STAGES]; /* profile used */
} adaptra_plan_info_t;

typedef struct adaptra_planner* adaptra_planner_t;
int adaptra_planner_create(const adaptra_planner_desc_t* d, adaptra_planner_t* out);
int adaptra_planner_destroy(adaptra_planner_t p);
/* Queue a new profile (e.g. adaptra_exec_profile's medians); ticks >= 1. */
int adaptra_planner_set_profile(adaptra_planner_t p, const int64_t* tF, const int64_t* tB, const int64_t* tW);
/* Plan the next iteration under link latencies c[S-1] (finite, >= 0; a failed
 * link is planned at its delegated-path cost, R33).  Outputs (each optional):
 * ops_out[S*3N] / n_ops_out[S] as adaptra_schedule, x_out[S], *replanned_out = 1
 * when x changed, info. */
int adaptra_planner_step(adaptra_planner_t p, const int64_t* c, adaptra_op_t* ops_out, int32_t* n_ops_out,
                         int32_t* x_out, int32_t* replanned_out, adaptra_plan_info_t* info);

/* ================================================================ GEMM
 * One dense contraction C[m,n] = sum_k A(m,k) B(n,k) over Z batches, with a
 * fused epilogue.  bf16 operands run on the tcgen05/TMEM/TMA kernel (fp32
 * accumulate in TMEM); fp32 operands run on the SIMT parity kernel.
 * This is the contraction behind stage F, B (dX) and W (dW).
 *
 * Addressing: A(m,k) of batch z is element
 *   A[(row(z) + r) * lda + col(z) + q],  (r,q) = (m,k) if a_mn == 0 (K-major)
 *                                        (r,q) = (k,m) if a_mn == 1 (MN-major)
 *   row(z) = z1*a_row1 + z2*a_row2, col(z) = z1*a_col1 + z2*a_col2,
 *   z1 = z / zdiv, z2 = z % zdiv.  a_rows x a_cols is the extent of the stored
 *   2-D matrix (reads outside it return 0).  Same for B with (n,k).
 * Output/aux/rowv are offset per batch by z1*x_1 + z2*x_2 elements.
 */
#define ADAPTRA_EPI_STORE 0     /* C = alpha*acc (+ bias[n])                               */
#define ADAPTRA_EPI_GELU 1      /* aux = acc + bias[n];  C = gelu(aux)       (R25)         */
#define ADAPTRA_EPI_RESID 2     /* C = acc + bias[n] + R[m,n]                              */
#define ADAPTRA_EPI_DGELU 3     /* C = acc * gelu'(aux[m,n])                               */
#define ADAPTRA_EPI_ACC_F32 4   /* Cf32[m,n] += alpha*acc   (deferred W accumulation)      */
#define ADAPTRA_EPI_STORE_F32 5 /* Cf32[m,n] = alpha*acc                                   */
#define ADAPTRA_EPI_DSOFTMAX 6  /* C = aux[m,n] * (acc - rowv[m]) * alpha  (softmax bwd)   */
/* C = acc (bf16) and, per 128-column head h and row m = s*T + t,
 * rowv[(s*H + h)*T + t] = sum_c bf16(C[m,c]) * aux[m,c]: the attention
 * backward's D = rowsum(dO o O) fused into the GEMM that produces dO
 * (rowv_1 = T tokens per sequence, rowv_2 = H heads; bf16, N % 256 == 0,
 * unbatched, the 2-CTA 256-wide tile path only). */
#define ADAPTRA_EPI_STORE_ROWDOT 7

#define ADAPTRA_CAUSAL_NONE 0
#define ADAPTRA_CAUSAL_TILE 1   /* skip output tiles strictly above the diagonal           */
#define ADAPTRA_CAUSAL_KEND 2   /* k < min(K, m_tile_end)                                  */
#define ADAPTRA_CAUSAL_KSTART 3 /* k >= m_tile_start                                       */

#define ADAPTRA_F32 0
#define ADAPTRA_BF16 1

typedef struct adaptra_gemm_desc {
  int32_t dtype; /* ADAPTRA_F32 | ADAPTRA_BF16 (A, B, C, aux, R element type; Cf32 always fp32) */
  int32_t M, N, K, Z, zdiv;
  const void* A;
  int64_t lda, a_rows, a_cols, a_row1, a_row2, a_col1, a_col2;
  int32_t a_mn, b_mn;
  const void* B;
  int64_t ldb, b_rows, b_cols, b_row1, b_row2, b_col1, b_col2;
  int32_t epi, causal;
  float alpha;
  int32_t pad0;
  void* C;
  int64_t ldc, c_1, c_2;
  void* aux;
  int64_t ldaux, aux_1, aux_2;
  const void* R;
  int64_t ldr;
  const float* bias;
  const float* rowv;
  int64_t rowv_1, rowv_2;
} adaptra_gemm_desc_t;

int adaptra_gemm(const adaptra_gemm_desc_t* g, void* stream);

/* Process-wide tuning knobs (take effect for launches after the call).
 * ADAPTRA_TUNE_GEMM_SMS: SMs a persistent tcgen05 GEMM launch may occupy
 * (rounded down to CTA pairs; 0 = all).  When several pipeline stages share a
 * GPU, a smaller grid leaves SMs to the other stages' kernels and gives each
 * CTA more tiles over which to pay its prologue and last epilogue. */
#define ADAPTRA_TUNE_GEMM_SMS 1
/* ADAPTRA_TUNE_ATTN_SMS: the same cap for the persistent attention forward. */
#define ADAPTRA_TUNE_ATTN_SMS 2
int adaptra_set_tuning(int32_t key, int64_t value);

/* Live kernel timing (bench roofline): when enabled, every tcgen05 GEMM launch
 * is bracketed by CUDA events on its own stream; kind 0 = the stage's linear
 * layers (unbatched), kind 2 = the batched attention products (materialised
 * fp32 path), kind 3 / 4 = the fused attention forward / backward.  collect() waits for
 * the recorded launches of `kind`, returns their count, summed duration (ms),
 * algorithmic FLOPs (2MNK per batch, causal products counted at 1/2, R28) and
 * operand/result bytes, and forgets them. */
int adaptra_prof_enable(int32_t on);
/* Number of this library's kernel launches in this process so far. */
int64_t adaptra_launch_count(void);
int adaptra_prof_collect(int32_t kind, int64_t* n_launches, double* sum_ms, double* flops, double* bytes);
/* Same, plus the union of the collected launches' [start, end) intervals
 * across all streams of the device (ms): the wall time during which at least
 * one launch of this kind was running.  With several stage streams on one GPU
 * launches overlap, so sum_ms / n overstates a launch's own duration. */
int adaptra_prof_collect_ex(int32_t kind, int64_t* n_launches, double* sum_ms, double* union_ms, double* flops,
                            double* bytes);

/* ================================================================ stage compute
 * One pipeline stage = n_layers identical blocks (R24/R19: uniform stages).
 * block MLP: y = x + gelu(x W1^T + b1) W2^T + b2                (config C0)
 * block GPT: GPT-2 pre-LN block (LN1, QKV, causal attention, O + residual,
 *            LN2, FC1 + GeLU, FC2 + residual)
 * Activations are row-major [b*T, d] in `dtype`.
 *
 * Parameter buffers (caller-owned, device):
 *  wts  (dtype): per layer, the GEMM matrices in [out, in] row-major order
 *        GPT: Wqkv[3d,d], Wo[d,d], W1[dff,d], W2[d,dff];  MLP: W1[dff,d], W2[d,dff]
 *  vecs (fp32):  per layer
 *        GPT: ln1_g[d], ln1_b[d], bqkv[3d], bo[d], ln2_g[d], ln2_b[d], b1[dff], b2[d]
 *        MLP: b1[dff], b2[d]
 *  gwts, gvecs (fp32): gradients, same layouts as wts / vecs; W ops accumulate
 *        into them (deferred weight gradients).
 *  stash (bytes = n_slots * adaptra_stage_slot_bytes): what W needs of one
 *        in-flight microbatch (GEMM inputs and output gradients); taken at F,
 *        freed at W (slot index chosen by the caller).
 *  stash_fb (bytes = n_slots_fb * adaptra_stage_slot_fb_bytes): what only B
 *        needs (qkv, attention probabilities, FC1 pre-activation); taken at F
 *        and freed at the end of B by the stage itself, in issue order
 *        ("B ... immediately free activation memory").
 *  work  (bytes = adaptra_stage_work_bytes): per-stage scratch (attention
 *        work buffers, the deterministic column-sum partials and tickets of
 *        W), reused by every op issued on the stage's stream.
 */
#define ADAPTRA_BLOCK_MLP 0
#define ADAPTRA_BLOCK_GPT 1

typedef struct adaptra_stage_desc {
  int32_t block, dtype;
  int32_t n_layers, d, d_ff, n_heads;
  int32_t b, T;            /* microbatch = b sequences of T tokens            */
  int32_t is_first, is_last;
  int32_t n_microbatches;  /* N: loss is L = (1/N) sum_j L_j (R19)           */
  int32_t n_slots;          /* F->W slots (caller-indexed)                    */
  int32_t n_slots_fb;       /* F->B slots (stage-managed free list)           */
  void* wts;
  float* vecs;
  float* gwts;
  float* gvecs;
  void* stash;
  void* stash_fb;
  void* work;
} adaptra_stage_desc_t;

typedef struct adaptra_stage* adaptra_stage_t;

int64_t adaptra_stage_slot_bytes(const adaptra_stage_desc_t* d);
int64_t adaptra_stage_slot_fb_bytes(const adaptra_stage_desc_t* d);
int64_t adaptra_stage_work_bytes(const adaptra_stage_desc_t* d);
int64_t adaptra_stage_wts_elems(const adaptra_stage_desc_t* d);
int64_t adaptra_stage_vecs_elems(const adaptra_stage_desc_t* d);
int adaptra_stage_create(const adaptra_stage_desc_t* d, adaptra_stage_t* out);
int adaptra_stage_destroy(adaptra_stage_t s);

/* F: forward of microbatch into stash slot `slot`.
 *  x_in   [b*T, d] dtype, must stay valid until W of this slot (mailbox slot).
 *  y_out  [b*T, d] dtype, written by the last GEMM epilogue (may be a peer
 *         mailbox mapped over NVLink); ignored on the last stage.
 *  target [b*T, d] fp32 (last stage only); loss_acc: fp32 scalar, += L_j / N
 *         (block partials summed in a fixed order: the loss is reproducible
 *         bit for bit, independent of scheduling and transport). */
int adaptra_stage_F(adaptra_stage_t s, int32_t slot, const void* x_in, void* y_out, const float* target,
                    float* loss_acc, void* stream);
/* B: input gradient only.  dy_in [b*T,d] dtype (NULL on the last
 * stage: the MSE seed from F is used); dx_out [b*T,d] dtype (ignored on the
 * first stage).  Keeps every GEMM's output gradient in the slot for W. */
int adaptra_stage_B(adaptra_stage_t s, int32_t slot, const void* dy_in, void* dx_out, void* stream);
/* W: weight gradients of the slot, accumulated
 * into gwts/gvecs (dW += dY^T X in fp32, db += sum dY, LN dgamma/dbeta). */
int adaptra_stage_W(adaptra_stage_t s, int32_t slot, void* stream);
/* W of two slots as one launch: every dW += X^T dY product runs over both
 * microbatches' rows (K = 2 b T, slot_a's rows first) and is reduce-added into
 * the fp32 gradient once (the executor uses it for two consecutive W ops of
 * a stage's order, $ADAPTRA_W_PAIRS=0 disables); bias / LN sums per slot. */
int adaptra_stage_W2(adaptra_stage_t s, int32_t slot_a, int32_t slot_b, void* stream);
/* The same for 1..4 slots (K = n b T, slots[0]'s rows first); the executor
 * groups up to $ADAPTRA_W_GROUP (default 4) consecutive W ops. */
int adaptra_stage_Wn(adaptra_stage_t s, const int32_t* slots, int32_t n, void* stream);
int adaptra_stage_zero_grads(adaptra_stage_t s, void* stream);

/* ================================================================ transport
 * One direction of one link (stage i -> i+1 for forward activations, i+1 -> i
 * for input gradients) is an inbox on the receiving stage and an
 * outbox on the sending stage.  One message of `bytes` per microbatch.
 *
 * Inbox (library-allocated so it can be exported over CUDA IPC):
 *   mailbox  [n_mb * bytes] device memory of the receiver, one slot per mb;
 *   flags    uint32[n_mb] in pinned, device-mapped HOST memory (a POSIX shm
 *            segment, so the sender's process can map it); message (mb) of
 *            iteration `epoch` is ready when flags[mb] >= epoch (epochs start
 *            at 1, increase; wrap-around compare);
 *   host ring (optional, POSIX shm `host_name`, pinned with cudaHostRegister):
 *            [n_mb * bytes] data + uint32[n_mb] host flags: the delegated path
 *            (P:2270-2350).  A process-wide delegate thread copies arrived host
 *            slots into the mailbox (H2D, copy engine) and posts the device flag.
 * Outbox (sender side):
 *   dst(mb)  where the producing kernel writes: the peer mailbox slot itself
 *            (DIRECT, mailbox on the same GPU: the last GEMM epilogue stores
 *            into it, no copy) or a local staging slot (DIRECT to another GPU:
 *            the copy engine moves it over NVLink on the outbox's stream --
 *            epilogue stores straight into peer memory measured 1.75x slower;
 *            P2P: a copy kernel moves it; HOST: D2H into the host ring).
 *   send     enqueues the transfer on the outbox's own stream after the
 *            producing op (never on the compute stream) and posts the flag.
 * Flags live in pinned, device-mapped host memory (POSIX shm, so they can be
 * mapped by the sender's process); a producer GPU posts a flag with a
 * one-thread system-scope release-store kernel after its data, the gate and
 * delegate threads post from the host, and the consuming stage's own host
 * thread waits on it (bounded by $ADAPTRA_TIMEOUT_MS, default 120 s) before
 * launching the consuming op -- the paper's busy wait.  Every
 * stage has its own thread, so a late message delays only the ops that follow
 * it in that stage's order (no cross-stage head-of-line blocking).
 * Latency injection (R16): with latency c > 0 the flag of each message is
 * posted c ns after its data is in place, by a process-wide gate thread that
 * polls the completion event (no SM use, messages pipeline).  Latency
 * ADAPTRA_LINK_DOWN marks the GPU path failed: the outbox switches to the
 * HOST path (the inbox must be told with adaptra_inbox_set_host); the
 * delegated path's own latency then applies.
 */
#define ADAPTRA_LINK_DIRECT 0
#define ADAPTRA_LINK_P2P 1
#define ADAPTRA_LINK_HOST 2
#define ADAPTRA_LINK_DOWN INT64_MAX
#define ADAPTRA_IPC_BYTES 128

typedef struct adaptra_inbox* adaptra_inbox_t;
typedef struct adaptra_outbox* adaptra_outbox_t;

/* host_name: NULL = no delegated path for this inbox. */
int adaptra_inbox_create(int32_t dev, int32_t n_mb, int64_t bytes, const char* host_name, adaptra_inbox_t* out);
int adaptra_inbox_destroy(adaptra_inbox_t ib);
/* 128 bytes: CUDA IPC handle of the mailbox (64) + name of the flag segment (64). */
int adaptra_inbox_export(adaptra_inbox_t ib, uint8_t* handle_out);
void* adaptra_inbox_slot(adaptra_inbox_t ib, int32_t mb);
/* Wait on the CALLING HOST THREAD until message mb of iteration epoch is in
 * the mailbox (its flag, in pinned host memory, reaches epoch; spin, then
 * yield, then 2 us sleeps; ELINK after $ADAPTRA_TIMEOUT_MS, default 120 s),
 * then return the slot address in slot_out.  `consumer` is unused: the caller
 * launches the consuming op on its stream after this returns, so stream order
 * puts the op after the data.  Only the stage thread that consumes the message
 * blocks (every stage has its own thread), so a late message delays only the
 * ops that follow it in that stage's order -- no cross-stage head-of-line
 * blocking; the paper's busy wait. */
int adaptra_recv(adaptra_inbox_t ib, int32_t mb, uint32_t epoch, void* consumer, void** slot_out);
/* Abort path: set every flag to 0x3F3F3F3F (>= any epoch) so that all host waiters proceed
 * (after a failed or timed-out iteration); adaptra_inbox_reset clears flags
 * (and host flags) back to 0 before epochs restart at 1. */
int adaptra_inbox_poison(adaptra_inbox_t ib);
int adaptra_inbox_reset(adaptra_inbox_t ib);
/* Receiver side of the delegated path on (1) / off (0). */
int adaptra_inbox_set_host(adaptra_inbox_t ib, int32_t on);

/* Same-process outbox (stages co-located in one process; devices may differ). */
int adaptra_outbox_open_local(int32_t dev, adaptra_inbox_t peer, int32_t mode, adaptra_outbox_t* out);
/* Cross-process outbox from an exported inbox handle (IPC over NVLink). */
int adaptra_outbox_open_ipc(int32_t dev, const uint8_t* handle, int32_t n_mb, int64_t bytes, const char* host_name,
                            int32_t mode, adaptra_outbox_t* out);
int adaptra_outbox_close(adaptra_outbox_t ob);
void* adaptra_outbox_dst(adaptra_outbox_t ob, int32_t mb);
/* Injected latency in ns (>= 0), or ADAPTRA_LINK_DOWN (delegated host path). */
int adaptra_set_link_latency(adaptra_outbox_t ob, int64_t latency_ns);
/* Delegation policy ("the delegated communication path is
 * activated only upon the detection of communication delays"): PATH_HOST sends
 * this outbox's messages over the delegated host path while the link is up
 * (its injected latency still applies: the slow network is on both paths);
 * PATH_GPU (default) uses the link's mode.  The receiving inbox must be told
 * with adaptra_inbox_set_host.  Set between iterations. */
#define ADAPTRA_PATH_GPU 0
#define ADAPTRA_PATH_HOST 1
int adaptra_link_set_path(adaptra_outbox_t ob, int32_t path);
/* The P2P link mode's transfer kernel (P:1575-1577 inter-stage activations /
 * gradients): copies `bytes` from `src` to `dst` (device pointers, either may
 * be a peer GPU's memory; peer access is enabled on first use) on `stream` with 16-byte
 * vector loads/stores from 32 CTAs (few SMs taken from compute); falls back to
 * cudaMemcpyAsync when not 16-byte aligned.  Exposed for transfer benchmarks. */
int adaptra_p2p_copy(void* dst, const void* src, int64_t bytes, void* stream);
/* Send message mb of iteration epoch once the work already enqueued on
 * `producer` (the producing op) has completed. */
int adaptra_send(adaptra_outbox_t ob, int32_t mb, void* producer, uint32_t epoch);
/* Host-blocking variants used by the in-order baseline (ADAPTRA_EXEC_INORDER):
 * block the calling thread until message mb of iteration epoch is in the
 * mailbox / has been delivered to the receiver (as a synchronous send/recv in
 * the compute sequence would). */
int adaptra_recv_blocking(adaptra_inbox_t ib, int32_t mb, uint32_t epoch, void** slot_out);
int adaptra_send_wait(adaptra_outbox_t ob, int32_t mb, uint32_t epoch);
/* Gate statistics since open: messages, sum/max of (flag post - data ready) in ns
 * (all cumulative since the outbox was opened). */
int adaptra_link_stats(adaptra_outbox_t ob, int64_t* n_msgs, int64_t* sum_delay_ns, int64_t* max_delay_ns);
/* Same, but the max covers only the messages since the previous _take (it is
 * reset to 0 by this call); n_msgs and sum_delay_ns stay cumulative. */
int adaptra_link_stats_take(adaptra_outbox_t ob, int64_t* n_msgs, int64_t* sum_delay_ns, int64_t* max_delay_ns);

/* ================================================================ executor
 * Interprets one iteration of a stage's op order (from adaptra_schedule) on
 * the stage's compute stream from a dedicated host thread: per op, a host
 * wait for its input message's flag (adaptra_recv; only this stage's thread
 * waits, so a late message never stalls another stage's launches: no HOL
 * stall), the F/B/W kernels, CUDA events around the op, and the
 * send of its output (adaptra_send: never blocks).  At most
 * $ADAPTRA_LOOKAHEAD (default 3) ops are queued ahead on the stream.  Stash
 * slots are taken at F and released at W (in op order, on the one compute
 * stream).
 */
typedef struct adaptra_exec_desc {
  adaptra_stage_t stage;
  int32_t stage_index, n_stages, n_microbatches;
  adaptra_inbox_t in_fwd;     /* activations from stage i-1 (NULL on stage 0)   */
  adaptra_inbox_t in_bwd;     /* gradients from stage i+1 (NULL on stage S-1)   */
  adaptra_outbox_t out_fwd;   /* to stage i+1 (NULL on stage S-1)               */
  adaptra_outbox_t out_bwd;   /* to stage i-1 (NULL on stage 0)                 */
  void* compute_stream;
  const void* const* inputs;   /* stage 0: n_mb device pointers [b*T, d]        */
  const float* const* targets; /* stage S-1: n_mb device pointers [b*T, d] fp32 */
  float* loss_acc;             /* stage S-1: device fp32 scalar                 */
} adaptra_exec_desc_t;

typedef struct adaptra_exec* adaptra_exec_t;

typedef struct adaptra_iter_stats {
  int64_t n_ops;
  int64_t busy_ns;          /* sum of op durations (CUDA events, compute stream) */
  int64_t first_start_ns;   /* relative to the iteration start event             */
  int64_t last_end_ns;
  int64_t op_ns[3];         /* summed duration per kind F, B, W                  */
  int64_t op_cnt[3];
  int64_t host_enqueue_ns;  /* host time spent enqueueing the iteration          */
} adaptra_iter_stats_t;

int adaptra_exec_create(const adaptra_exec_desc_t* d, adaptra_exec_t* out);
int adaptra_exec_destroy(adaptra_exec_t e);
/* Post one iteration: ops[n] (kind, mb) in order; flags: ADAPTRA_MERGE_W runs W
 * right after each B (1F1B); ADAPTRA_EXEC_INORDER is the sequential-launch
 * baseline that exhibits head-of-line blocking: every receive
 * blocks the stage thread until its message is there, and a send blocks it
 * while more than Q of the outbox's messages are undelivered (the
 * transmission queue is full; Q = $ADAPTRA_INORDER_QUEUE,
 * default 2; 0 = rendezvous, every send waits for its delivery + c).
 * Non-blocking (the stage thread enqueues). */
#define ADAPTRA_EXEC_INORDER 16u
int adaptra_run_iteration(adaptra_exec_t e, const adaptra_op_t* ops, int32_t n, uint32_t epoch, uint32_t flags);
/* N4 host activation offload ("offloading activation and
 * gradients to the host lifts the GPU memory pressure").  The
 * stage's n_slots device F->W stash slots may be fewer than the microbatches
 * in flight: host_pool (caller-owned pinned memory, n_host_slots x
 * adaptra_stage_slot_bytes) takes the overflow.  Per iteration the executor
 * plans from the known op order (Belady): when an F finds no free device
 * slot, the complete slot (its B done) whose W is furthest away is spilled --
 * the D2H is issued on an offload stream right after that slot's B, and the F
 * waits only for that copy -- and a spilled slot is prefetched (H2D) when a
 * device slot is free and its W is within `window` ops (default 4), or at the
 * latest right before its W, which waits for it.  Results are bit-identical
 * to the all-device run.  ENOMEM from adaptra_run_iteration's stage thread
 * when even the host pool cannot hold the order's demand.  n_host_slots = 0
 * disables. */
int adaptra_exec_set_offload(adaptra_exec_t e, void* host_pool, int32_t n_host_slots, int32_t window);
/* The executor's offload plan for one stage's op order, as a pure host
 * function (what adaptra_run_iteration plans internally): n_dev device slots,
 * n_host host slots, flags ADAPTRA_MERGE_W.  slot_out[n] = device slot each op
 * uses; actions_out[cap][6] = {spill (1) / prefetch (0), mb, device slot, host
 * slot, issued after op q, awaited by op q'}; *n_actions_out = total.
 * ENOMEM when the order cannot run in n_dev + n_host slots. */
int adaptra_offload_plan(const adaptra_op_t* ops, int32_t n, int32_t N, int32_t n_dev, int32_t n_host, int32_t window,
                         uint32_t flags, int32_t* slot_out, int32_t* actions_out, int32_t cap, int32_t* n_actions_out);
/* Spills and prefetches planned for the last iteration; bytes moved since creation. */
int adaptra_exec_offload_stats(adaptra_exec_t e, int32_t* n_spill, int32_t* n_prefetch, int64_t* bytes);

/* ---------------------------------------------------------------- NCCL baseline (N1)
 * north_star: "NCCL send/recv is used only as the baseline".  With
 * ADAPTRA_EXEC_NCCL the executor runs the fixed execution plan of
 * Megatron-style runtimes: per op, in order on the compute
 * stream, the previous op's send grouped with this op's receive
 * (ncclSend/ncclRecv inside ncclGroupStart/End), then the op's kernels; an
 * injected latency c (adaptra_set_link_latency on the outbox) holds the compute
 * stream for c before the send -- a slow transfer blocks everything queued
 * behind it (head-of-line blocking).  A failed link costs
 * `down_ns` (the measured delegated-path time) instead.  Outputs go to the
 * sender's staging slots, inputs land in the receiver's mailbox slots; the
 * epoch flags are not used.  One communicator over all ranks (one stage per
 * GPU: NCCL refuses two ranks on one device). */
#define ADAPTRA_NCCL_ID_BYTES 128
#define ADAPTRA_EXEC_NCCL 32u
/* ncclGetUniqueId into id_out[128] (rank 0; broadcast it to the others). */
int adaptra_nccl_unique_id(uint8_t* id_out);
/* ncclCommInitRank on device dev; *comm_out is an ncclComm_t. */
int adaptra_nccl_comm_init(const uint8_t* id, int32_t nranks, int32_t rank, int32_t dev, void** comm_out);
int adaptra_nccl_comm_destroy(void* comm);
/* One ncclSend (send != 0) or ncclRecv of `bytes` at device `buf` with NCCL
 * rank `peer` on `stream` (a cudaStream_t; NULL = legacy stream).  Used by
 * the binding's buffering probe (R39). */
int adaptra_nccl_p2p(void* comm, int32_t send, void* buf, int64_t bytes, int32_t peer, void* stream);
/* Communicator and the NCCL ranks of stages i-1 / i+1 (-1 if none). */
int adaptra_exec_set_nccl(adaptra_exec_t e, void* comm, int32_t rank_prev, int32_t rank_next, int64_t down_ns);
/* Receive-posting plan (R39).  Blocking send/recv groups deadlock once a
 * link's NCCL buffers are full: orders with many warm-up forwards (Alg. 2's
 * adapted orders, the greedy ZB orders) have stage i blocked sending to i+1
 * while i+1 is blocked sending to i.  The paper's adaptation assumes no such
 * stalls (Sec. 5 intro).  Stage i's group p is issued before op p's
 * kernels (p = n_ops[i]: the trailing flush) and holds op p-1's send plus the
 * receives of the ops q with post_at[q] == p.  A send completes once its
 * receive is posted, or on its own while fewer than `buffered` earlier
 * messages of the link are unreceived (0 = strict rendezvous).  From
 * post_at[q] = q (-1 for ops without a receive) the plan simulates the groups
 * of all S stages and, whenever none can proceed, moves the oldest unreceived
 * message's receive into the receiver's current group (the receive's mailbox
 * slot is its microbatch's own, so posting early is safe) -- only where the
 * buffers cannot absorb the orders.  ops: the S orders back to back (stage
 * i's n_ops[i] ops after stage i-1's), post_at_out the same layout.  EPLAN if
 * the send and receive orders of a link differ or the orders violate
 * dependencies. */
int adaptra_nccl_post_plan(int32_t S, const adaptra_op_t* ops, const int32_t* n_ops, uint32_t flags,
                           int32_t buffered, int32_t* post_at_out);
/* Stage's slice of that plan for the NEXT iteration only (n = its op count;
 * without it each receive is posted with its own op).  EINVAL at run time if
 * it does not fit the orders. */
int adaptra_exec_set_nccl_post(adaptra_exec_t e, const int32_t* post_at, int32_t n);

/* End-to-end host I/O (NULL disables): on stage 0, host_inputs[n_mb] are pinned
 * host buffers of `bytes` each; every iteration copies them into the device
 * inputs of the exec desc (H2D on a side stream, issued in the order stage 0
 * runs its F ops; F(mb) waits for its own copy), so the input upload overlaps
 * the pipeline.  On the last stage, host_loss receives the iteration's loss
 * (D2H behind the last op).  Caller-owned; must outlive the iterations. */
int adaptra_exec_set_host_io(adaptra_exec_t e, const void* const* host_inputs, int64_t bytes, float* host_loss);
/* Report op times relative to `event` (a cudaEvent_t recorded by the caller on
 * the stage's device before the iteration; NULL = the stage's own start
 * event), so that stages sharing a device share one time base. */
int adaptra_exec_set_time_base(adaptra_exec_t e, void* event);
/* Wait until the stage thread has enqueued the whole iteration; returns its
 * error, if any (call on every stage before adaptra_exec_wait so that a
 * failed stage can be detected and the others released). */
int adaptra_exec_join(adaptra_exec_t e);
/* Wait until the iteration's GPU work on this stage is complete (bounded by
 * $ADAPTRA_TIMEOUT_MS, default 120000: ELINK on timeout); fill stats.
 * op_times_out (optional, n x 2 int64: start, end ns) gets per-op times. */
int adaptra_exec_wait(adaptra_exec_t e, adaptra_iter_stats_t* stats_out, int64_t* op_times_out);

/* Profiler ("the profiler continuously tracks ...", P:2436-2437
 * "leverages CUDA Events"): every adaptra_exec_wait appends the iteration's
 * mean op time per kind (F, B, W; CUDA events on the compute stream) to the
 * stage's history (last 256 iterations).  t_out[3] = for each kind the lower
 * median over the last k iterations that ran that kind, floored to `quantum`
 * ns and at least one quantum (0 if none ran), i.e. the t^F_i, t^B_i, t^W_i
 * ticks the planner takes.  EINVAL if k < 1 or quantum < 1. */
int adaptra_exec_profile(adaptra_exec_t e, int32_t k, int64_t quantum, int64_t* t_out);
/* The reduction it applies: lower median of v[n], floored to quantum, >= quantum
 * (-1 on bad arguments).  Pure host function. */
int64_t adaptra_median_ticks(const int64_t* v, int32_t n, int64_t quantum);

#ifdef __cplusplus
}
#endif
#endif /* ADAPTRA_H */
