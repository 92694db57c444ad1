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
 *    stash arenas, workspaces and pinned host rings are caller-owned (the
 *    Python binding allocates them with torch); the library only borrows raw
 *    pointers.  Only opaque handles (stage, link) are library-allocated and
 *    are freed by the matching *_destroy / *_close call.
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

/* Number of dependency/completeness violations of a timed schedule (0 = valid). */
int adaptra_validate(int32_t S, int32_t N, const int64_t* tF, const int64_t* tB, const int64_t* tW,
                     const int64_t* c, const adaptra_op_t* ops, const int32_t* n_ops, uint32_t flags,
                     int32_t* n_violations_out);

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
 *  stash (bytes = n_slots * adaptra_stage_slot_bytes): saved activations of
 *        one in-flight microbatch per slot; F fills slot s, B reads it and adds
 *        output gradients, W consumes and frees it.
 *  work  (bytes = adaptra_stage_work_bytes): per-stage scratch (attention
 *        scores), reused by every op issued on the stage's stream.
 */
#define ADAPTRA_BLOCK_MLP 0
#define ADAPTRA_BLOCK_GPT 1

typedef struct adaptra_stage_desc {
  int32_t block, dtype;
  int32_t n_layers, d, d_ff, n_heads;
  int32_t b, T;            /* microbatch = b sequences of T tokens            */
  int32_t is_first, is_last;
  int32_t n_microbatches;  /* N: loss is L = (1/N) sum_j L_j (R19)           */
  int32_t n_slots;
  void* wts;
  float* vecs;
  float* gwts;
  float* gvecs;
  void* stash;
  void* work;
} adaptra_stage_desc_t;

typedef struct adaptra_stage* adaptra_stage_t;

int64_t adaptra_stage_slot_bytes(const adaptra_stage_desc_t* d);
int64_t adaptra_stage_work_bytes(const adaptra_stage_desc_t* d);
int64_t adaptra_stage_wts_elems(const adaptra_stage_desc_t* d);
int64_t adaptra_stage_vecs_elems(const adaptra_stage_desc_t* d);
int adaptra_stage_create(const adaptra_stage_desc_t* d, adaptra_stage_t* out);
int adaptra_stage_destroy(adaptra_stage_t s);

/* F: forward of microbatch into stash slot `slot`.
 *  x_in   [b*T, d] dtype, must stay valid until W of this slot (mailbox slot).
 *  y_out  [b*T, d] dtype, written by the last GEMM epilogue (may be a peer
 *         mailbox mapped over NVLink); ignored on the last stage.
 *  target [b*T, d] fp32 (last stage only); loss_acc: fp32 scalar, += L_j / N. */
int adaptra_stage_F(adaptra_stage_t s, int32_t slot, const void* x_in, void* y_out, const float* target,
                    float* loss_acc, void* stream);
/* B: input gradient only.  dy_in [b*T,d] dtype (NULL on the last
 * stage: the MSE seed from F is used); dx_out [b*T,d] dtype (ignored on the
 * first stage).  Keeps every GEMM's output gradient in the slot for W. */
int adaptra_stage_B(adaptra_stage_t s, int32_t slot, const void* dy_in, void* dx_out, void* stream);
/* W: weight gradients of the slot, accumulated
 * into gwts/gvecs (dW += dY^T X in fp32, db += sum dY, LN dgamma/dbeta). */
int adaptra_stage_W(adaptra_stage_t s, int32_t slot, void* stream);
int adaptra_stage_zero_grads(adaptra_stage_t s, void* stream);

/* ================================================================ transport
 * A link carries stage i's F output to stage i+1 (dir FWD) and stage i+1's B
 * output to stage i (dir BWD), one message of `bytes` per microbatch.
 * Receiver-side mailboxes: one slot per microbatch per direction.  Readiness
 * is a per-(dir, mb) 32-bit flag equal to the iteration epoch.
 *
 * Modes:
 *  ADAPTRA_LINK_DIRECT  producer epilogue writes straight into the receiver
 *                       mailbox (same device or NVLink peer pointer); send
 *                       only posts the flag.
 *  ADAPTRA_LINK_P2P     send runs the P2P copy kernel (src -> peer mailbox
 *                       over NVLink), then posts the flag.
 *  ADAPTRA_LINK_HOST    delegated path: D2H copy engine into a
 *                       pinned host slot on a side stream, then H2D into the
 *                       receiver mailbox, then the flag.  Also the path taken
 *                       while the link is down (latency ADAPTRA_LINK_DOWN).
 * Latency injection: adaptra_set_link_latency(l, c) delays the flag of every
 * later message by c ns after the producing op completes (a pure per-message
 * latency, R16), applied by a host gate thread with no SM use.
 */
#define ADAPTRA_LINK_DIRECT 0
#define ADAPTRA_LINK_P2P 1
#define ADAPTRA_LINK_HOST 2
#define ADAPTRA_DIR_FWD 0
#define ADAPTRA_DIR_BWD 1
#define ADAPTRA_LINK_DOWN INT64_MAX

typedef struct adaptra_link_desc {
  int32_t mode;
  int32_t n_mb;            /* mailbox slots per direction                     */
  int64_t bytes;           /* message size                                    */
  int32_t dev_up, dev_down;/* CUDA device of stage i and of stage i+1         */
  /* Receiver mailboxes, [n_mb * bytes] each, on the receiving device (caller
   * owned; may be IPC-mapped peer pointers).  fwd_mbox lives on dev_down,
   * bwd_mbox on dev_up. */
  void* fwd_mbox;
  void* bwd_mbox;
  /* Flags: uint32[n_mb] each, device memory of the receiver (fwd_flags on
   * dev_down, bwd_flags on dev_up), zero-initialised by the caller. */
  uint32_t* fwd_flags;
  uint32_t* bwd_flags;
  /* Delegated path: pinned host staging [n_mb * bytes] per direction (may be NULL
   * unless mode == HOST or the link can go down). */
  void* host_fwd;
  void* host_bwd;
} adaptra_link_desc_t;

typedef struct adaptra_link* adaptra_link_t;

int adaptra_link_open(const adaptra_link_desc_t* d, adaptra_link_t* out);
int adaptra_link_close(adaptra_link_t l);
/* Injected latency in ns (>= 0), or ADAPTRA_LINK_DOWN: the link's GPU path has
 * failed and traffic moves to the delegated host path. */
int adaptra_set_link_latency(adaptra_link_t l, int64_t latency_ns);
/* Send message (dir, mb) of iteration `epoch`: src is the producer's buffer
 * (NULL in DIRECT mode: data already in the mailbox).  `produced` is a
 * cudaEvent_t recorded after the producing op on the producer stream; the
 * send is enqueued on the link's own streams, never on the compute stream. */
int adaptra_send(adaptra_link_t l, int32_t dir, int32_t mb, const void* src, void* produced, uint32_t epoch);
/* Make `consumer` stream wait (on the GPU, no host blocking) until message
 * (dir, mb) of iteration `epoch` is in the mailbox; returns its address. */
int adaptra_recv(adaptra_link_t l, int32_t dir, int32_t mb, void* consumer, uint32_t epoch, void** slot_out);
/* Achieved per-message latency statistics since open (ns). */
int adaptra_link_stats(adaptra_link_t l, int64_t* n_msgs, int64_t* sum_latency_ns, int64_t* max_latency_ns);

/* ================================================================ executor
 * Interprets one iteration of a stage's op list (from adaptra_schedule) on the
 * stage's compute stream: per op, wait for its input message on the GPU
 * (never blocking the host, so no HOL stall: P:1801-1828), launch the F/B/W
 * kernels, record CUDA events, and hand the output to the link.
 */
typedef struct adaptra_exec_desc {
  adaptra_stage_t stage;
  int32_t stage_index, n_stages, n_microbatches;
  adaptra_link_t link_up;     /* link to stage i-1 (NULL on the first stage)  */
  adaptra_link_t link_down;   /* link to stage i+1 (NULL on the last stage)   */
  void* compute_stream;
  /* first stage: microbatch inputs, n_mb pointers [b*T,d] dtype (device) */
  const void* const* inputs;
  /* last stage: targets, n_mb pointers [b*T,d] fp32 (device) */
  const float* const* targets;
  float* loss_acc;            /* device fp32 scalar                            */
  uint32_t merge_w;           /* 1F1B: run W right after B                     */
} adaptra_exec_desc_t;

typedef struct adaptra_exec* adaptra_exec_t;

typedef struct adaptra_iter_stats {
  int64_t n_ops;
  int64_t busy_ns;           /* sum of op durations on the compute stream (CUDA events) */
  int64_t first_start_ns;    /* relative to the iteration's time base         */
  int64_t last_end_ns;
  int64_t op_ns[3];          /* summed duration per kind F, B, W              */
  int64_t op_cnt[3];
} adaptra_iter_stats_t;

int adaptra_exec_create(const adaptra_exec_desc_t* d, adaptra_exec_t* out);
int adaptra_exec_destroy(adaptra_exec_t e);
/* Enqueue one iteration: ops[n] in order (kind, mb); slots are assigned from
 * the stage's stash pool in op order (F takes, W frees).  Non-blocking. */
int adaptra_run_iteration(adaptra_exec_t e, const adaptra_op_t* ops, int32_t n, uint32_t epoch, void* t0_event);
/* Block until the iteration's work on this stage is done; fill stats. */
int adaptra_exec_wait(adaptra_exec_t e, adaptra_iter_stats_t* stats_out);

#ifdef __cplusplus
}
#endif
#endif /* ADAPTRA_H */
