// Per-stage schedule executor: one host thread per stage interprets the
// stage's op order for one iteration.  Before an op that consumes a message
// the stage's thread waits on the message's flag in pinned host memory
// (adaptra_recv); every stage has its own thread, so a late message delays
// only the ops after it in that stage's order and never another stage's
// launches (no cross-stage head-of-line blocking).  Outputs are
// handed to the outbox right after the producing op (adaptra_send, never
// blocks).  ADAPTRA_EXEC_INORDER (bounded send queue) and ADAPTRA_EXEC_NCCL
// (NCCL send/recv in the compute sequence, receives posted per the R39 plan)
// are the blocking baselines (N1).  Per-kind op times feed the profiler
// (adaptra_exec_profile, a1).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <array>
#include <deque>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../../include/adaptra.h"
#include "../comm/transport.h"
#include "../util.h"

namespace adaptra {
int stage_n_slots(adaptra_stage_t s);
int stage_device(adaptra_stage_t s);
void* stage_slot_base(adaptra_stage_t s, int slot);
int64_t stage_slot_nbytes(adaptra_stage_t s);
void stage_get_meta(adaptra_stage_t s, int slot, const void** x_in, const void** dy_in);
void stage_set_meta(adaptra_stage_t s, int to, int from, const void* x_in, const void* dy_in);
}  // namespace adaptra

using namespace adaptra;

static const bool g_dbg = getenv("ADAPTRA_DEBUG") != nullptr;
#define DBG(...)                                  \
  do {                                            \
    if (g_dbg) {                                  \
      fprintf(stderr, "[exec %d] ", d.stage_index); \
      fprintf(stderr, __VA_ARGS__);               \
      fprintf(stderr, "\n");                      \
    }                                             \
  } while (0)

namespace adaptra {
// N4 stash offload: the F->W stash slots of a
// stage live in D device slots; with a host pool of H slots, slots whose W is
// far in the op order are spilled there after their B and prefetched back
// before their W, so the stage can hold more in-flight microbatches than fit
// in HBM.  The plan is static per iteration (the order is known in advance):
// Belady eviction (the complete slot whose W is furthest away) when an F
// needs a slot, the spill D2H issued right after the victim's B, the prefetch
// H2D up to `window` ops ahead of its W when a device slot is free (and the
// F ops before that W leave one), at the latest right before the W.
int offload_plan(const adaptra_op_t* ops, int n, int N, int D, int H, int window, bool merge, SlotPlan& P) {
  P.slot.assign(n, -1);
  P.after.assign(n, {});
  P.wait.assign(n, {});
  P.n_spill = P.n_prefetch = 0;
  std::vector<int> bpos(N + 1, INT32_MAX), wpos(N + 1, INT32_MAX), state(N + 1, 0), dsl(N + 1, -1), hsl(N + 1, -1);
  for (int q = n - 1; q >= 0; --q) {
    const int mb = ops[q].mb;
    if (mb < 1 || mb > N || ops[q].kind < 0 || ops[q].kind > 2) return set_error(ADAPTRA_EINVAL, "exec: bad op");
    if (ops[q].kind == ADAPTRA_OP_B) bpos[mb] = q;
    if (ops[q].kind == ADAPTRA_OP_W || (merge && ops[q].kind == ADAPTRA_OP_B)) wpos[mb] = q;
  }
  std::vector<int> free_dev;
  // free host slots with the issue position of the prefetch that freed them:
  // every copy runs in issue order on one offload stream, so a spill may
  // reuse a host slot only if it is issued at or after that prefetch
  std::vector<std::pair<int, int>> free_host;
  for (int k = D - 1; k >= 0; --k) free_dev.push_back(k);
  for (int k = H - 1; k >= 0; --k) free_host.push_back({k, -1});
  int next_id = 0;
  auto evict = [&](int q, int keep) -> int {
    int best = -1;
    for (int mb = 1; mb <= N; ++mb)
      if (state[mb] == 1 && mb != keep && bpos[mb] < q && wpos[mb] > q && (best < 0 || wpos[mb] > wpos[best]))
        best = mb;
    if (best < 0) return set_error(ADAPTRA_ENOMEM, "exec: stash slots exhausted (no complete slot to offload)");
    if (free_host.empty()) return set_error(ADAPTRA_ENOMEM, "exec: stash slots exhausted (host offload pool full)");
    size_t hk = 0;  // the host slot free the longest
    for (size_t k = 1; k < free_host.size(); ++k)
      if (free_host[k].second < free_host[hk].second) hk = k;
    const int h = free_host[hk].first;
    // issued right after the victim's B, or after the prefetch that freed h
    // (always <= q - 1: every prefetch planned so far is issued by then)
    const int at = std::max(bpos[best], free_host[hk].second);
    free_host.erase(free_host.begin() + hk);
    OffAct a{1, best, dsl[best], h, dsl[best], next_id++};
    P.after[at].push_back(a);
    P.wait[q].push_back(a.id);
    P.n_spill++;
    state[best] = 2;
    hsl[best] = h;
    free_dev.push_back(dsl[best]);
    return ADAPTRA_OK;
  };
  auto prefetch = [&](int mb, int after_q, int w_q) {
    const int s = free_dev.back();
    free_dev.pop_back();
    OffAct a{0, mb, s, hsl[mb], -1, next_id++};
    P.after[after_q].push_back(a);
    P.wait[w_q].push_back(a.id);
    P.n_prefetch++;
    free_host.push_back({hsl[mb], after_q});
    state[mb] = 1;
    dsl[mb] = s;
  };
  for (int q = 0; q < n; ++q) {
    const adaptra_op_t& o = ops[q];
    const int mb = o.mb;
    if (o.kind == ADAPTRA_OP_F) {
      if (state[mb] != 0) return set_error(ADAPTRA_EINVAL, "exec: F twice");
      int rc;
      if (free_dev.empty() && (rc = evict(q, -1))) return rc;
      dsl[mb] = free_dev.back();
      free_dev.pop_back();
      state[mb] = 1;
      P.slot[q] = dsl[mb];
    } else {
      if (state[mb] == 0) return set_error(ADAPTRA_EINVAL, o.kind == ADAPTRA_OP_B ? "exec: B before F" : "exec: W before F");
      if (state[mb] == 2) {  // W of a spilled slot not prefetched yet: fetch now
        int rc;
        if (free_dev.empty() && (rc = evict(q, mb))) return rc;
        if (q == 0) return set_error(ADAPTRA_EINVAL, "exec: W first");
        prefetch(mb, q - 1, q);
      }
      P.slot[q] = dsl[mb];
      if (o.kind == ADAPTRA_OP_W || merge) {
        free_dev.push_back(dsl[mb]);
        state[mb] = 0;
      }
    }
    // early prefetch: the spilled slot with the nearest W, if it is within
    // `window` ops and the F ops before it leave a device slot free
    while (H > 0 && !free_dev.empty()) {
      int nb = -1;
      for (int m = 1; m <= N; ++m)
        if (state[m] == 2 && (nb < 0 || wpos[m] < wpos[nb])) nb = m;
      if (nb < 0 || wpos[nb] > q + window) break;
      int nf = 0;
      for (int r = q + 1; r < wpos[nb]; ++r) nf += ops[r].kind == ADAPTRA_OP_F;
      if ((int)free_dev.size() <= nf) break;
      prefetch(nb, q, wpos[nb]);
    }
  }
  return ADAPTRA_OK;
}
}  // namespace adaptra

extern "C" int adaptra_offload_plan(const adaptra_op_t* ops, int32_t n, int32_t N, int32_t n_dev, int32_t n_host,
                                    int32_t window, uint32_t flags, int32_t* slot_out, int32_t* actions_out,
                                    int32_t cap, int32_t* n_actions_out) {
  if (!ops || n < 0 || N < 1 || n_dev < 1 || n_host < 0 || !slot_out || cap < 0 || (cap > 0 && !actions_out) ||
      !n_actions_out)
    return set_error(ADAPTRA_EINVAL, "offload_plan: bad args");
  adaptra::SlotPlan P;
  int rc = adaptra::offload_plan(ops, n, N, n_dev, n_host, window > 0 ? window : 4, flags & ADAPTRA_MERGE_W, P);
  if (rc) return rc;
  for (int q = 0; q < n; ++q) slot_out[q] = P.slot[q];
  int k = 0;
  for (int q = 0; q < n; ++q)
    for (const auto& a : P.after[q]) {
      if (k < cap) {
        int32_t* r = actions_out + 6 * k;
        r[0] = a.spill;
        r[1] = a.mb;
        r[2] = a.dslot;
        r[3] = a.hslot;
        r[4] = q;  // issued right after op q
        int w = -1;
        for (int t = 0; t < n && w < 0; ++t)
          for (int id : P.wait[t])
            if (id == a.id) w = t;
        r[5] = w;  // the op that waits for it
      }
      ++k;
    }
  *n_actions_out = k;
  return ADAPTRA_OK;
}

// NCCL arm receive-posting plan (R39).  Group p of stage i is issued before
// op p's kernels (p = n_i: the trailing flush) and holds the send of op p-1's
// output plus the receives of every op q with post_at[q] == p; a group ends
// when all of its operations have completed.  A send completes once its
// receive is posted, or on its own while fewer than `buffered` earlier
// messages of its link sit unreceived in NCCL's buffers (0: strict
// rendezvous); a receive completes once posted and its send has completed.
// Starting from post_at[q] = q, whenever no stream can move, the oldest
// unreceived message of a link whose sender is blocked has its receive
// hoisted into the receiver's current group -- the receive's mailbox slot is
// its microbatch's own, so posting early is safe -- until every stream ends.
extern "C" int adaptra_nccl_post_plan(int32_t S, const adaptra_op_t* ops, const int32_t* n_ops, uint32_t flags,
                                      int32_t buffered, int32_t* post_at_out) {
  if (S < 1 || !ops || !n_ops || !post_at_out || buffered < 0)
    return set_error(ADAPTRA_EINVAL, "nccl_post_plan: bad args");
  const bool merge = flags & ADAPTRA_MERGE_W;
  std::vector<int64_t> off(S + 1, 0);
  for (int i = 0; i < S; ++i) {
    if (n_ops[i] < 0) return set_error(ADAPTRA_EINVAL, "nccl_post_plan: bad n_ops");
    off[i + 1] = off[i] + n_ops[i];
  }
  // channels: 2i = forward activations i -> i+1, 2i+1 = gradients i+1 -> i
  struct End {
    int stage, op, mb;
  };
  const int n_ch = 2 * std::max(0, S - 1);
  std::vector<std::vector<End>> snd(n_ch), rcv(n_ch);
  std::vector<int> r_ch(off[S], -1), r_k(off[S], -1), s_ch(off[S], -1), s_k(off[S], -1);
  for (int i = 0; i < S; ++i)
    for (int q = 0; q < n_ops[i]; ++q) {
      const adaptra_op_t& o = ops[off[i] + q];
      const int64_t g = off[i] + q;
      int rc_ = -1, sc = -1;
      if (o.kind == ADAPTRA_OP_F) {
        if (i > 0) rc_ = 2 * (i - 1);
        if (i < S - 1) sc = 2 * i;
      } else if (o.kind == ADAPTRA_OP_B) {
        if (i < S - 1) rc_ = 2 * i + 1;
        if (i > 0) sc = 2 * (i - 1) + 1;
      } else if (o.kind != ADAPTRA_OP_W || merge) {
        return set_error(ADAPTRA_EPLAN, "nccl_post_plan: bad op kind");
      }
      if (rc_ >= 0) {
        r_ch[g] = rc_;
        r_k[g] = (int)rcv[rc_].size();
        rcv[rc_].push_back({i, q, o.mb});
      }
      if (sc >= 0) {
        s_ch[g] = sc;
        s_k[g] = (int)snd[sc].size();
        snd[sc].push_back({i, q, o.mb});
      }
    }
  for (int ch = 0; ch < n_ch; ++ch) {
    if (snd[ch].size() != rcv[ch].size()) return set_error(ADAPTRA_EPLAN, "nccl_post_plan: send/recv counts differ");
    for (size_t k = 0; k < snd[ch].size(); ++k)
      if (snd[ch][k].mb != rcv[ch][k].mb)
        return set_error(ADAPTRA_EPLAN, "nccl_post_plan: send and receive orders differ on a link");
  }
  for (int i = 0; i < S; ++i)
    for (int q = 0; q < n_ops[i]; ++q) post_at_out[off[i] + q] = r_ch[off[i] + q] >= 0 ? q : -1;
  // ns / nr: sends / receives of each link completed so far (both complete in
  // link order: one stream issues them in that order)
  std::vector<int> pos(S, 0), ns(n_ch, 0), nr(n_ch, 0);
  auto posted = [&](const End& b) { return pos[b.stage] == post_at_out[off[b.stage] + b.op]; };
  auto complete = [&](int i, int p) {
    if (p > 0) {
      const int64_t g = off[i] + p - 1;
      if (s_ch[g] >= 0 && ns[s_ch[g]] <= s_k[g]) return false;
    }
    for (int q = p; q < n_ops[i]; ++q) {
      const int64_t g = off[i] + q;
      if (post_at_out[g] == p && nr[r_ch[g]] <= r_k[g]) return false;
    }
    return true;
  };
  for (;;) {
    bool progress = false, finished = true;
    for (int ch = 0; ch < n_ch; ++ch) {
      for (bool moved = true; moved;) {
        moved = false;
        const int k = ns[ch];
        if (k < (int)snd[ch].size() && pos[snd[ch][k].stage] == snd[ch][k].op + 1 &&
            (k - nr[ch] < buffered || (nr[ch] == k && posted(rcv[ch][k])))) {
          ++ns[ch];
          moved = true;
        }
        if (nr[ch] < ns[ch] && posted(rcv[ch][nr[ch]])) {
          ++nr[ch];
          moved = true;
        }
        progress |= moved;
      }
    }
    for (int i = 0; i < S; ++i) {
      while (pos[i] <= n_ops[i] && complete(i, pos[i])) {
        ++pos[i];
        progress = true;
      }
      if (pos[i] <= n_ops[i]) finished = false;
    }
    if (finished) return ADAPTRA_OK;
    if (progress) continue;
    // no stream can move: hoist the oldest unreceived message of the first
    // link whose sender is blocked on it
    bool hoisted = false;
    for (int ch = 0; ch < n_ch && !hoisted; ++ch) {
      const int k = ns[ch];
      if (k >= (int)snd[ch].size() || pos[snd[ch][k].stage] != snd[ch][k].op + 1) continue;
      const End& b = rcv[ch][nr[ch]];
      int32_t& pa = post_at_out[off[b.stage] + b.op];
      if (pa > pos[b.stage]) {
        pa = pos[b.stage];
        hoisted = true;
      }
    }
    if (!hoisted) return set_error(ADAPTRA_EPLAN, "nccl_post_plan: receives wait on unposted sends (orders violate dependencies)");
  }
}

struct adaptra_exec {
  adaptra_exec_desc_t d{};
  int dev = 0;
  cudaStream_t cs = nullptr;
  std::thread th;
  std::mutex mu;
  std::condition_variable cv;
  bool stop = false, has_job = false, busy = false;
  std::vector<adaptra_op_t> ops;
  uint32_t epoch = 0, flags = 0;
  int rc = ADAPTRA_OK;
  std::string err;
  int64_t host_ns = 0;
  cudaEvent_t ev_t0 = nullptr;
  cudaEvent_t ev_base = nullptr;  // optional common time base (same device), set by the caller
  std::vector<cudaEvent_t> ev_s, ev_e;
  // a1 profiler: per completed iteration, the mean op time per kind (ns; -1 = none)
  std::deque<std::array<int64_t, 3>> hist;
  // host I/O (end-to-end runs): stage 0 copies each microbatch's input from
  // pinned host memory (H2D on its own stream, overlapped with compute; F(mb)
  // waits for its copy); the last stage copies the loss back at the end
  const void* const* host_inputs = nullptr;
  int64_t host_in_bytes = 0;
  float* host_loss = nullptr;
  cudaStream_t h2d = nullptr;
  std::vector<cudaEvent_t> ev_in;
  // N4 stash offload: the F->W stash slots of the
  // stage live in `n_slots` device slots; with a pinned host pool, slots whose
  // W is far in the op order are spilled there after their B and prefetched
  // back before their W, so the stage can hold more in-flight microbatches
  // than fit in HBM.  The plan is static per iteration (the op order is known
  // in advance): Belady eviction (the complete slot whose W is furthest away)
  // when an F needs a slot, spill D2H issued right after the victim's B,
  // prefetch H2D up to `pf_window` ops ahead of its W when a slot is free.
  adaptra::SlotPlan P;
  char* host_pool = nullptr;
  int n_host = 0, pf_window = 4;
  cudaStream_t off = nullptr;
  std::vector<cudaEvent_t> ev_act;
  std::vector<std::pair<const void*, const void*>> saved_meta;  // per mb (x_in, dy_in) while spilled
  int64_t spilled_bytes = 0;

  int plan_slots() {
    int rc = adaptra::offload_plan(ops.data(), (int)ops.size(), d.n_microbatches, stage_n_slots(d.stage), n_host,
                                   pf_window, flags & ADAPTRA_MERGE_W, P);
    if (rc) return rc;
    const int n_act = P.n_spill + P.n_prefetch;
    if (n_act > (int)ev_act.size()) {
      cudaSetDevice(dev);
      const size_t old = ev_act.size();
      ev_act.resize(n_act);
      for (size_t k = old; k < ev_act.size(); ++k)
        ADAPTRA_CUDA_TRY(cudaEventCreateWithFlags(&ev_act[k], cudaEventDisableTiming));
    }
    if (n_act > 0 && !off) return set_error(ADAPTRA_EINVAL, "exec: offload planned without a host pool");
    saved_meta.assign(d.n_microbatches + 1, {nullptr, nullptr});
    from_slot_of.assign(d.n_microbatches + 1, -1);
    return ADAPTRA_OK;
  }

  // before op q's kernels: wait for the spills / prefetches it depends on
  int pre_op(size_t q) {
    for (int id : P.wait[q]) ADAPTRA_CUDA_TRY(cudaStreamWaitEvent(cs, ev_act[id], 0));
    return ADAPTRA_OK;
  }

  // after op q has been enqueued: issue the offload copies planned there
  int post_op(size_t q) {
    if (P.after[q].empty()) return ADAPTRA_OK;
    const int64_t sb = stage_slot_nbytes(d.stage);
    ADAPTRA_CUDA_TRY(cudaStreamWaitEvent(off, ev_e[q], 0));
    for (const OffAct& a : P.after[q]) {
      char* hp = host_pool + (size_t)a.hslot * sb;
      char* dp = (char*)stage_slot_base(d.stage, a.dslot);
      if (a.spill) {
        const void *x = nullptr, *y = nullptr;
        stage_get_meta(d.stage, a.dslot, &x, &y);
        saved_meta[a.mb] = {x, y};
        from_slot_of[a.mb] = a.dslot;
        ADAPTRA_CUDA_TRY(cudaMemcpyAsync(hp, dp, sb, cudaMemcpyDeviceToHost, off));
      } else {
        stage_set_meta(d.stage, a.dslot, from_slot_of[a.mb], saved_meta[a.mb].first, saved_meta[a.mb].second);
        ADAPTRA_CUDA_TRY(cudaMemcpyAsync(dp, hp, sb, cudaMemcpyHostToDevice, off));
      }
      spilled_bytes += sb;
      ADAPTRA_CUDA_TRY(cudaEventRecord(ev_act[a.id], off));
    }
    return ADAPTRA_OK;
  }
  std::vector<int> from_slot_of;

  // NCCL baseline arm (N1): communicator and the peers' ranks
  void* nccl = nullptr;
  int nccl_prev = -1, nccl_next = -1;
  int64_t nccl_down_ns = 0;

  // ADAPTRA_EXEC_NCCL: the fixed execution plan of Megatron-style runtimes
  // (P:1801-1813).  Per op, in order on the compute stream: one group
  // (ncclGroupStart/End) with the send of the previous op's output and the
  // receive of this op's input (as send_forward_recv_backward pairs them),
  // then the op's kernels.  nccl_post (adaptra_exec_set_nccl_post, one-shot)
  // moves receives into earlier groups where strict rendezvous would
  // otherwise deadlock (R39).  An injected latency c holds the stream for c
  // before the send (the transfer occupies the in-order stream,
  // P:1815-1828); a failed link costs its measured delegated-path time
  // instead (baselines have no delegation, so this is generous to them).
  std::vector<int32_t> nccl_post;
  int run_nccl() {
    const int S = d.n_stages, i = d.stage_index, N = d.n_microbatches;
    const bool merge = flags & ADAPTRA_MERGE_W;
    const size_t n = ops.size();
    int rc;
    auto has_recv = [&](size_t q) {
      return (ops[q].kind == ADAPTRA_OP_F && i > 0) || (ops[q].kind == ADAPTRA_OP_B && i < S - 1);
    };
    // at[p]: the ops whose receives group p posts
    std::vector<std::vector<int>> at(n + 1);
    const bool planned = nccl_post.size() == n;
    for (size_t q = 0; q < n; ++q) {
      const int p = planned ? nccl_post[q] : (has_recv(q) ? (int)q : -1);
      if (has_recv(q) != (p >= 0) || p > (int)q)
        return set_error(ADAPTRA_EINVAL, "exec: NCCL receive plan does not fit these orders");
      if (p >= 0) at[p].push_back((int)q);
    }
    nccl_post.clear();
    adaptra::P2POp pend{1, nullptr, 0, -1};
    int64_t p_lat = 0;
    std::vector<adaptra::P2POp> grp;
    auto issue = [&](size_t p) -> int {
      grp.clear();
      if (pend.buf) {
        if (p_lat > 0) {
          int r = stream_spin(cs, p_lat);
          if (r) return r;
        }
        grp.push_back(pend);
        pend.buf = nullptr;
      }
      for (int q : at[p]) {
        const int m = ops[q].mb;
        if (m < 1 || m > N) return set_error(ADAPTRA_EINVAL, "exec: bad microbatch");
        if (ops[q].kind == ADAPTRA_OP_F)
          grp.push_back({0, adaptra_inbox_slot(d.in_fwd, m - 1), outbox_bytes(d.out_bwd), nccl_prev});
        else
          grp.push_back({0, adaptra_inbox_slot(d.in_bwd, m - 1), outbox_bytes(d.out_fwd), nccl_next});
      }
      return nccl_p2p(nccl, grp.data(), (int)grp.size(), cs);
    };
    auto lat_of = [&](adaptra_outbox_t ob) {
      int64_t l = outbox_latency(ob);
      return l == ADAPTRA_LINK_DOWN ? nccl_down_ns : l;
    };
    for (size_t q = 0; q < n; ++q) {
      if (q > 0 && (rc = post_op(q - 1))) return rc;
      const adaptra_op_t& o = ops[q];
      const int mb = o.mb;
      if (mb < 1 || mb > N) return set_error(ADAPTRA_EINVAL, "exec: bad microbatch");
      const int slot = P.slot[q];
      if (o.kind != ADAPTRA_OP_F && o.kind != ADAPTRA_OP_B && o.kind != ADAPTRA_OP_W)
        return set_error(ADAPTRA_EINVAL, "exec: bad op kind");
      if (o.kind != ADAPTRA_OP_F && slot < 0) return set_error(ADAPTRA_EINVAL, "exec: B/W before F");
      if ((rc = pre_op(q))) return rc;
      if (o.kind == ADAPTRA_OP_F && i == 0 && host_inputs)
        ADAPTRA_CUDA_TRY(cudaStreamWaitEvent(cs, ev_in[mb - 1], 0));
      if ((rc = issue(q))) return rc;
      if (o.kind == ADAPTRA_OP_F) {
        const void* x = i == 0 ? d.inputs[mb - 1] : adaptra_inbox_slot(d.in_fwd, mb - 1);
        void* y = (i < S - 1) ? outbox_local_slot(d.out_fwd, mb - 1) : nullptr;
        if (i < S - 1 && !y) return set_error(ADAPTRA_ENOMEM, "exec: no send buffer");
        ADAPTRA_CUDA_TRY(cudaEventRecord(ev_s[q], cs));
        if ((rc = adaptra_stage_F(d.stage, slot, x, y, i == S - 1 ? d.targets[mb - 1] : nullptr,
                                  i == S - 1 ? d.loss_acc : nullptr, cs)))
          return rc;
        ADAPTRA_CUDA_TRY(cudaEventRecord(ev_e[q], cs));
        if (i < S - 1) {
          pend = {1, y, outbox_bytes(d.out_fwd), nccl_next};
          p_lat = lat_of(d.out_fwd);
        }
      } else if (o.kind == ADAPTRA_OP_B) {
        void* dy = i < S - 1 ? adaptra_inbox_slot(d.in_bwd, mb - 1) : nullptr;
        void* dx = (i > 0) ? outbox_local_slot(d.out_bwd, mb - 1) : nullptr;
        if (i > 0 && !dx) return set_error(ADAPTRA_ENOMEM, "exec: no send buffer");
        ADAPTRA_CUDA_TRY(cudaEventRecord(ev_s[q], cs));
        if ((rc = adaptra_stage_B(d.stage, slot, dy, dx, cs))) return rc;
        if (merge) {
          if ((rc = adaptra_stage_W(d.stage, slot, cs))) return rc;
        }
        ADAPTRA_CUDA_TRY(cudaEventRecord(ev_e[q], cs));
        if (i > 0) {
          pend = {1, dx, outbox_bytes(d.out_bwd), nccl_prev};
          p_lat = lat_of(d.out_bwd);
        }
      } else {
        ADAPTRA_CUDA_TRY(cudaEventRecord(ev_s[q], cs));
        if ((rc = adaptra_stage_W(d.stage, slot, cs))) return rc;
        ADAPTRA_CUDA_TRY(cudaEventRecord(ev_e[q], cs));
      }
    }
    if (n > 0 && (rc = post_op(n - 1))) return rc;
    return issue(n);
  }

  int run_one() {
    cudaSetDevice(dev);
    const int S = d.n_stages, i = d.stage_index, N = d.n_microbatches;
    const bool merge = flags & ADAPTRA_MERGE_W;
    const bool inorder = flags & ADAPTRA_EXEC_INORDER;
    // In-order baseline (N1): a send blocks the stage thread only
    // while more than Q of this outbox's messages are still undelivered (the
    // transmission queue is full); Q = $ADAPTRA_INORDER_QUEUE (default 2;
    // 0 = synchronous rendezvous, every send waits for its delivery)
    static const int qdepth = [] {
      const char* v = getenv("ADAPTRA_INORDER_QUEUE");
      return v ? std::max(0, atoi(v)) : 2;
    }();
    std::deque<std::pair<int, uint32_t>> q_fwd, q_bwd;
    auto send_q = [&](adaptra_outbox_t ob, std::deque<std::pair<int, uint32_t>>& qu, int m) -> int {
      qu.emplace_back(m, epoch);
      while ((int)qu.size() > qdepth) {
        int r = adaptra_send_wait(ob, qu.front().first, qu.front().second);
        if (r) return r;
        qu.pop_front();
      }
      return ADAPTRA_OK;
    };
    const int64_t t_start = now_ns();
    int rc;
    if ((rc = plan_slots())) return rc;
    ADAPTRA_CUDA_TRY(cudaEventRecord(ev_t0, cs));
    if (i == S - 1 && d.loss_acc) ADAPTRA_CUDA_TRY(cudaMemsetAsync(d.loss_acc, 0, sizeof(float), cs));
    if (i == 0 && host_inputs) {
      // the iteration's inputs, in the order stage 0 consumes them
      ADAPTRA_CUDA_TRY(cudaStreamWaitEvent(h2d, ev_t0, 0));
      for (const adaptra_op_t& o : ops) {
        if (o.kind != ADAPTRA_OP_F || o.mb < 1 || o.mb > N) continue;
        ADAPTRA_CUDA_TRY(cudaMemcpyAsync((void*)d.inputs[o.mb - 1], host_inputs[o.mb - 1], host_in_bytes,
                                         cudaMemcpyHostToDevice, h2d));
        ADAPTRA_CUDA_TRY(cudaEventRecord(ev_in[o.mb - 1], h2d));
      }
    }
    DBG("start epoch %u n_ops %zu", epoch, ops.size());
    if ((rc = adaptra_stage_zero_grads(d.stage, cs))) return rc;  // gradients of this iteration only
    DBG("zeroed");
    if (flags & ADAPTRA_EXEC_NCCL) {
      if (!nccl) return set_error(ADAPTRA_EINVAL, "exec: NCCL arm without a communicator (adaptra_exec_set_nccl)");
      if ((rc = run_nccl())) return rc;
      if (i == S - 1 && host_loss && d.loss_acc)
        ADAPTRA_CUDA_TRY(cudaMemcpyAsync(host_loss, d.loss_acc, sizeof(float), cudaMemcpyDeviceToHost, cs));
      host_ns = now_ns() - t_start;
      return ADAPTRA_OK;
    }
    // consecutive W ops per launch: $ADAPTRA_W_GROUP (1..4, default 4);
    // ADAPTRA_W_PAIRS=0 (the round-2 pair switch) means 1
    static const int w_group = [] {
      const char* g = getenv("ADAPTRA_W_GROUP");
      const char* p = getenv("ADAPTRA_W_PAIRS");
      int v = g ? atoi(g) : 4;
      if (p && atoi(p) == 0) v = 1;
      return std::max(1, std::min(4, v));
    }();
    static const int lookahead = [] {
      const char* v = getenv("ADAPTRA_LOOKAHEAD");
      return v ? atoi(v) : 3;
    }();
    for (size_t q = 0; q < ops.size(); ++q) {
      if (q > 0 && (rc = post_op(q - 1))) return rc;
      const adaptra_op_t& o = ops[q];
      const int mb = o.mb;
      DBG("op %zu kind %d mb %d", q, o.kind, o.mb);
      // bounded run-ahead: keep at most `lookahead` ops queued on the stream so
      // the launch queue stays shallow (waits on this stage's own work only)
      if ((int)q >= lookahead) {
        cudaEvent_t prev = ev_e[q - lookahead];
        while (cudaEventQuery(prev) == cudaErrorNotReady) std::this_thread::sleep_for(std::chrono::microseconds(5));
        cudaGetLastError();
      }
      if (mb < 1 || mb > N) return set_error(ADAPTRA_EINVAL, "exec: bad microbatch");
      if (o.kind == ADAPTRA_OP_F) {
        const int slot = P.slot[q];
        if ((rc = pre_op(q))) return rc;
        const void* x = nullptr;
        if (i == 0) {
          x = d.inputs[mb - 1];
          if (host_inputs) ADAPTRA_CUDA_TRY(cudaStreamWaitEvent(cs, ev_in[mb - 1], 0));
        } else {
          void* p = nullptr;
          if ((rc = inorder ? adaptra_recv_blocking(d.in_fwd, mb - 1, epoch, &p)
                            : adaptra_recv(d.in_fwd, mb - 1, epoch, cs, &p)))
            return rc;
          x = p;
        }
        void* y = (i < S - 1) ? adaptra_outbox_dst(d.out_fwd, mb - 1) : nullptr;
        ADAPTRA_CUDA_TRY(cudaEventRecord(ev_s[q], cs));
        DBG("  F recv done x=%p y=%p", x, y);
        if ((rc = adaptra_stage_F(d.stage, slot, x, y, i == S - 1 ? d.targets[mb - 1] : nullptr,
                                  i == S - 1 ? d.loss_acc : nullptr, cs)))
          return rc;
        DBG("  F launched");
        ADAPTRA_CUDA_TRY(cudaEventRecord(ev_e[q], cs));
        if (i < S - 1 && (rc = adaptra_send(d.out_fwd, mb - 1, cs, epoch))) return rc;
        if (inorder && i < S - 1 && (rc = send_q(d.out_fwd, q_fwd, mb - 1))) return rc;
      } else if (o.kind == ADAPTRA_OP_B) {
        const int slot = P.slot[q];
        if (slot < 0) return set_error(ADAPTRA_EINVAL, "exec: B before F");
        if ((rc = pre_op(q))) return rc;
        void* dy = nullptr;
        if (i < S - 1 && (rc = inorder ? adaptra_recv_blocking(d.in_bwd, mb - 1, epoch, &dy)
                                       : adaptra_recv(d.in_bwd, mb - 1, epoch, cs, &dy)))
          return rc;
        void* dx = (i > 0) ? adaptra_outbox_dst(d.out_bwd, mb - 1) : nullptr;
        ADAPTRA_CUDA_TRY(cudaEventRecord(ev_s[q], cs));
        DBG("  B recv done dy=%p dx=%p", dy, dx);
        if ((rc = adaptra_stage_B(d.stage, slot, dy, dx, cs))) return rc;
        DBG("  B launched");
        if (merge) {
          if ((rc = adaptra_stage_W(d.stage, slot, cs))) return rc;
        }
        ADAPTRA_CUDA_TRY(cudaEventRecord(ev_e[q], cs));
        if (i > 0 && (rc = adaptra_send(d.out_bwd, mb - 1, cs, epoch))) return rc;
        if (inorder && i > 0 && (rc = send_q(d.out_bwd, q_bwd, mb - 1))) return rc;
      } else if (o.kind == ADAPTRA_OP_W) {
        const int slot = P.slot[q];
        if (slot < 0) return set_error(ADAPTRA_EINVAL, "exec: W before F");
        if ((rc = pre_op(q))) return rc;
        // up to w_group consecutive W ops of the order run as one launch over
        // K = n bT (adaptra_stage_Wn): same work, one fp32 gradient
        // read-modify-write per group; the group's time is booked on its
        // first op (the others get zero length).  Not across offload copies:
        // a later W's slot may be refilled right after an earlier one frees it.
        int32_t grp[4] = {slot, 0, 0, 0};
        int n_grp = 1;
        while (!merge && n_grp < w_group && q + n_grp < ops.size() && ops[q + n_grp].kind == ADAPTRA_OP_W &&
               P.slot[q + n_grp] >= 0 && P.after[q + n_grp - 1].empty()) {
          const int32_t sl = P.slot[q + n_grp];
          bool dup = false;
          for (int k = 0; k < n_grp; ++k) dup = dup || grp[k] == sl;
          if (dup) break;
          grp[n_grp++] = sl;
        }
        if (n_grp > 1) {
          for (int k = 1; k < n_grp; ++k)
            if ((rc = pre_op(q + k))) return rc;
          ADAPTRA_CUDA_TRY(cudaEventRecord(ev_s[q], cs));
          if ((rc = adaptra_stage_Wn(d.stage, grp, n_grp, cs))) return rc;
          ADAPTRA_CUDA_TRY(cudaEventRecord(ev_e[q], cs));
          for (int k = 1; k < n_grp; ++k) {
            ADAPTRA_CUDA_TRY(cudaEventRecord(ev_s[q + k], cs));
            ADAPTRA_CUDA_TRY(cudaEventRecord(ev_e[q + k], cs));
            if ((rc = post_op(q + k - 1))) return rc;
          }
          q += n_grp - 1;
          continue;
        }
        ADAPTRA_CUDA_TRY(cudaEventRecord(ev_s[q], cs));
        if ((rc = adaptra_stage_W(d.stage, slot, cs))) return rc;
        ADAPTRA_CUDA_TRY(cudaEventRecord(ev_e[q], cs));
      } else {
        return set_error(ADAPTRA_EINVAL, "exec: bad op kind");
      }
    }
    if (!ops.empty() && (rc = post_op(ops.size() - 1))) return rc;
    if (i == S - 1 && host_loss && d.loss_acc)
      ADAPTRA_CUDA_TRY(cudaMemcpyAsync(host_loss, d.loss_acc, sizeof(float), cudaMemcpyDeviceToHost, cs));
    host_ns = now_ns() - t_start;
    DBG("enqueued all");
    return ADAPTRA_OK;
  }

  void loop() {
    for (;;) {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return stop || has_job; });
      if (stop) return;
      has_job = false;
      lk.unlock();
      int r = run_one();
      std::string e = r ? last_error() : "";
      lk.lock();
      rc = r;
      err = e;
      busy = false;
      cv.notify_all();
    }
  }
};

extern "C" int adaptra_exec_create(const adaptra_exec_desc_t* d, adaptra_exec_t* out) {
  if (!d || !out || !d->stage || d->n_stages < 1 || d->stage_index < 0 || d->stage_index >= d->n_stages ||
      d->n_microbatches < 1 || !d->compute_stream)
    return set_error(ADAPTRA_EINVAL, "exec_create: bad args");
  const int i = d->stage_index, S = d->n_stages;
  if ((i > 0 && (!d->in_fwd || !d->out_bwd)) || (i < S - 1 && (!d->in_bwd || !d->out_fwd)) ||
      (i == 0 && !d->inputs) || (i == S - 1 && (!d->targets || !d->loss_acc)))
    return set_error(ADAPTRA_EINVAL, "exec_create: missing link or io buffers");
  auto* e = new adaptra_exec();
  e->d = *d;
  e->cs = (cudaStream_t)d->compute_stream;
  e->dev = stage_device(d->stage);
  cudaSetDevice(e->dev);
  int cap = 3 * d->n_microbatches;
  e->ev_s.resize(cap);
  e->ev_e.resize(cap);
  cudaEventCreate(&e->ev_t0);
  for (int k = 0; k < cap; ++k) {
    cudaEventCreate(&e->ev_s[k]);
    cudaEventCreate(&e->ev_e[k]);
  }
  e->th = std::thread([e] { e->loop(); });
  *out = e;
  return ADAPTRA_OK;
}

extern "C" int adaptra_exec_destroy(adaptra_exec_t e) {
  if (!e) return ADAPTRA_OK;
  {
    std::unique_lock<std::mutex> lk(e->mu);
    e->cv.wait(lk, [&] { return !e->busy; });
    e->stop = true;
  }
  e->cv.notify_all();
  e->th.join();
  cudaSetDevice(e->dev);
  if (e->h2d) cudaStreamDestroy(e->h2d);
  if (e->off) cudaStreamDestroy(e->off);
  for (auto ev : e->ev_act) cudaEventDestroy(ev);
  for (auto ev : e->ev_in) cudaEventDestroy(ev);
  cudaEventDestroy(e->ev_t0);
  for (auto ev : e->ev_s) cudaEventDestroy(ev);
  for (auto ev : e->ev_e) cudaEventDestroy(ev);
  delete e;
  return ADAPTRA_OK;
}

extern "C" int adaptra_run_iteration(adaptra_exec_t e, const adaptra_op_t* ops, int32_t n, uint32_t epoch,
                                     uint32_t flags) {
  if (!e || !ops || n < 0 || n > (int)e->ev_s.size()) return set_error(ADAPTRA_EINVAL, "run_iteration: bad args");
  std::unique_lock<std::mutex> lk(e->mu);
  if (e->busy) return set_error(ADAPTRA_EINVAL, "run_iteration: previous iteration still running");
  e->ops.assign(ops, ops + n);
  if (!(flags & ADAPTRA_EXEC_NCCL)) e->nccl_post.clear();
  e->epoch = epoch;
  e->flags = flags;
  e->has_job = true;
  e->busy = true;
  e->rc = ADAPTRA_OK;
  e->cv.notify_all();
  return ADAPTRA_OK;
}

extern "C" int adaptra_exec_set_host_io(adaptra_exec_t e, const void* const* host_inputs, int64_t bytes,
                                        float* host_loss) {
  if (!e) return set_error(ADAPTRA_EINVAL, "exec_set_host_io: null");
  std::unique_lock<std::mutex> lk(e->mu);
  if (e->busy) return set_error(ADAPTRA_EINVAL, "exec_set_host_io: iteration running");
  const int i = e->d.stage_index, S = e->d.n_stages, N = e->d.n_microbatches;
  if (host_inputs && (i != 0 || bytes <= 0)) return set_error(ADAPTRA_EINVAL, "exec_set_host_io: inputs on stage 0 only");
  if (host_loss && i != S - 1) return set_error(ADAPTRA_EINVAL, "exec_set_host_io: loss on the last stage only");
  cudaSetDevice(e->dev);
  if (host_inputs && !e->h2d) {
    ADAPTRA_CUDA_TRY(cudaStreamCreateWithFlags(&e->h2d, cudaStreamNonBlocking));
    e->ev_in.resize(N);
    for (auto& ev : e->ev_in) ADAPTRA_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  e->host_inputs = host_inputs;
  e->host_in_bytes = bytes;
  e->host_loss = host_loss;
  return ADAPTRA_OK;
}

extern "C" int adaptra_exec_set_offload(adaptra_exec_t e, void* host_pool, int32_t n_host_slots, int32_t window) {
  if (!e || n_host_slots < 0 || (n_host_slots > 0 && !host_pool)) return set_error(ADAPTRA_EINVAL, "exec_set_offload: bad args");
  std::unique_lock<std::mutex> lk(e->mu);
  if (e->busy) return set_error(ADAPTRA_EINVAL, "exec_set_offload: iteration running");
  cudaSetDevice(e->dev);
  if (n_host_slots > 0 && !e->off) ADAPTRA_CUDA_TRY(cudaStreamCreateWithFlags(&e->off, cudaStreamNonBlocking));
  e->host_pool = (char*)host_pool;
  e->n_host = n_host_slots;
  e->pf_window = window > 0 ? window : 4;
  return ADAPTRA_OK;
}

extern "C" int adaptra_exec_offload_stats(adaptra_exec_t e, int32_t* n_spill, int32_t* n_prefetch, int64_t* bytes) {
  if (!e) return set_error(ADAPTRA_EINVAL, "exec_offload_stats: null");
  std::unique_lock<std::mutex> lk(e->mu);
  if (n_spill) *n_spill = e->P.n_spill;
  if (n_prefetch) *n_prefetch = e->P.n_prefetch;
  if (bytes) *bytes = e->spilled_bytes;
  return ADAPTRA_OK;
}

extern "C" int adaptra_exec_set_nccl(adaptra_exec_t e, void* comm, int32_t rank_prev, int32_t rank_next,
                                     int64_t down_ns) {
  if (!e) return set_error(ADAPTRA_EINVAL, "exec_set_nccl: null");
  std::unique_lock<std::mutex> lk(e->mu);
  if (e->busy) return set_error(ADAPTRA_EINVAL, "exec_set_nccl: iteration running");
  e->nccl = comm;
  e->nccl_prev = rank_prev;
  e->nccl_next = rank_next;
  e->nccl_down_ns = down_ns;
  return ADAPTRA_OK;
}

extern "C" int adaptra_exec_set_nccl_post(adaptra_exec_t e, const int32_t* post_at, int32_t n) {
  if (!e || n < 0 || (n > 0 && !post_at)) return set_error(ADAPTRA_EINVAL, "exec_set_nccl_post: bad args");
  std::unique_lock<std::mutex> lk(e->mu);
  if (e->busy) return set_error(ADAPTRA_EINVAL, "exec_set_nccl_post: iteration running");
  e->nccl_post.assign(post_at, post_at + n);
  return ADAPTRA_OK;
}

extern "C" int adaptra_exec_set_time_base(adaptra_exec_t e, void* event) {
  if (!e) return set_error(ADAPTRA_EINVAL, "exec_set_time_base: null");
  e->ev_base = (cudaEvent_t)event;
  return ADAPTRA_OK;
}

extern "C" int adaptra_exec_join(adaptra_exec_t e) {
  if (!e) return set_error(ADAPTRA_EINVAL, "exec_join: null");
  std::unique_lock<std::mutex> lk(e->mu);
  e->cv.wait(lk, [&] { return !e->busy; });
  if (e->rc) return set_error(e->rc, e->err);
  return ADAPTRA_OK;
}

extern "C" int adaptra_exec_wait(adaptra_exec_t e, adaptra_iter_stats_t* st, int64_t* op_times) {
  if (!e) return set_error(ADAPTRA_EINVAL, "exec_wait: null");
  {
    std::unique_lock<std::mutex> lk(e->mu);
    e->cv.wait(lk, [&] { return !e->busy; });
    if (e->rc) return set_error(e->rc, e->err);
  }
  cudaSetDevice(e->dev);
  // bounded wait: a message that never arrives must not hang the process
  static const int64_t timeout_ns = [] {
    const char* v = getenv("ADAPTRA_TIMEOUT_MS");
    return (v ? atoll(v) : 120000) * 1000000LL;
  }();
  const int64_t t0 = now_ns();
  for (;;) {
    cudaError_t q = cudaStreamQuery(e->cs);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) return set_error(ADAPTRA_ECUDA, std::string("exec_wait: ") + cudaGetErrorString(q));
    if (now_ns() - t0 > timeout_ns) return set_error(ADAPTRA_ELINK, "exec_wait: iteration timed out (message lost?)");
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
  adaptra_iter_stats_t s{};
  s.n_ops = (int64_t)e->ops.size();
  s.first_start_ns = INT64_MAX;
  s.last_end_ns = 0;
  for (size_t q = 0; q < e->ops.size(); ++q) {
    float a = 0.f, b = 0.f;
    cudaEvent_t base = e->ev_base ? e->ev_base : e->ev_t0;
    ADAPTRA_CUDA_TRY(cudaEventElapsedTime(&a, base, e->ev_s[q]));
    ADAPTRA_CUDA_TRY(cudaEventElapsedTime(&b, base, e->ev_e[q]));
    int64_t s0 = (int64_t)(a * 1e6), e0 = (int64_t)(b * 1e6);
    if (op_times) {
      op_times[2 * q] = s0;
      op_times[2 * q + 1] = e0;
    }
    s.busy_ns += e0 - s0;
    int k = e->ops[q].kind;
    if (k >= 0 && k < 3) {
      s.op_ns[k] += e0 - s0;
      s.op_cnt[k] += 1;
    }
    if (s0 < s.first_start_ns) s.first_start_ns = s0;
    if (e0 > s.last_end_ns) s.last_end_ns = e0;
  }
  if (s.n_ops == 0) s.first_start_ns = 0;
  s.host_enqueue_ns = e->host_ns;
  if (st) *st = s;
  std::array<int64_t, 3> m{-1, -1, -1};
  for (int k = 0; k < 3; ++k)
    if (s.op_cnt[k] > 0) m[k] = s.op_ns[k] / s.op_cnt[k];
  e->hist.push_back(m);
  while (e->hist.size() > 256) e->hist.pop_front();
  return ADAPTRA_OK;
}

extern "C" int64_t adaptra_median_ticks(const int64_t* v, int32_t n, int64_t quantum) {
  if (!v || n < 1 || quantum < 1) return -1;
  std::vector<int64_t> a(v, v + n);
  std::sort(a.begin(), a.end());
  const int64_t med = a[(n - 1) / 2];                  // lower median
  return std::max<int64_t>(quantum, med / quantum * quantum);  // floor to the quantum, >= 1 quantum
}

extern "C" int adaptra_exec_profile(adaptra_exec_t e, int32_t k, int64_t quantum, int64_t* t_out) {
  if (!e || k < 1 || quantum < 1 || !t_out) return set_error(ADAPTRA_EINVAL, "exec_profile: bad args");
  for (int kind = 0; kind < 3; ++kind) {
    std::vector<int64_t> v;
    for (auto it = e->hist.rbegin(); it != e->hist.rend() && (int)v.size() < k; ++it)
      if ((*it)[kind] >= 0) v.push_back((*it)[kind]);
    t_out[kind] = v.empty() ? 0 : adaptra_median_ticks(v.data(), (int32_t)v.size(), quantum);
  }
  return ADAPTRA_OK;
}
