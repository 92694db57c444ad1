// Host scheduling core: Alg. 1 GetInitWarmupFwds, Alg. 2 GetAdaptedWarmupFwds,
// Eq. 1, Alg. 3 SelectOp + Alg. 4 Schedule (discrete-time simulation), fixed-
// order replay and validation.  Pure int64 code, reentrant, no allocation
// outside std::vector.  Readings R1-R12 as in DESIGN.md §3.
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../../include/adaptra.h"
#include "../util.h"

namespace {

using adaptra::set_error;

bool valid_plan(int S, int N, const int32_t* x) {
  for (int i = 0; i + 1 < S; ++i)
    if (x[i] < x[i + 1]) return false;
  return x[S - 1] >= 1 && x[0] <= N;
}

int64_t ceil_div(int64_t a, int64_t b) {  // b > 0
  return a >= 0 ? (a + b - 1) / b : -((-a) / b);
}

struct Avail {
  int32_t kind, mb;
  int64_t ready;
};

struct StageSim {
  int32_t x_rem, x_orig;
  std::vector<Avail> avail;
  int64_t end = 0;
  int32_t nF = 0, nB = 0;
};

const int kPri[3] = {2, 3, 1};  // F:2, B:3, W:1

// Alg. 3 SelectOp.  Returns index into st.avail or -1.
int select_op(StageSim& st, int64_t t, bool cap) {
  int best = -1;
  if (st.x_rem > 0) {
    // Warm-up: only F, lowest microbatch (R6); None if no F is available.
    for (int k = 0; k < (int)st.avail.size(); ++k) {
      const Avail& a = st.avail[k];
      if (a.ready <= t && a.kind == ADAPTRA_OP_F && (best < 0 || a.mb < st.avail[best].mb)) best = k;
    }
    if (best >= 0) st.x_rem -= 1;
    return best;
  }
  const bool f_ok = !cap || (st.nF - st.nB < st.x_orig);
  for (int k = 0; k < (int)st.avail.size(); ++k) {
    const Avail& a = st.avail[k];
    if (a.ready > t) continue;
    if (a.kind == ADAPTRA_OP_F && !f_ok) continue;
    if (best < 0) {
      best = k;
      continue;
    }
    const Avail& b = st.avail[best];
    if (kPri[a.kind] > kPri[b.kind] || (kPri[a.kind] == kPri[b.kind] && a.mb < b.mb)) best = k;
  }
  return best;
}

struct Dur {
  std::vector<int64_t> d[3];
  Dur(int S, const int64_t* tF, const int64_t* tB, const int64_t* tW, bool merge) {
    for (int k = 0; k < 3; ++k) d[k].resize(S);
    for (int i = 0; i < S; ++i) {
      d[ADAPTRA_OP_F][i] = tF[i];
      d[ADAPTRA_OP_B][i] = tB[i] + (merge ? tW[i] : 0);
      d[ADAPTRA_OP_W][i] = tW[i];
    }
  }
};

// Dependencies of (i, kind, mb) (R8): up to 2 entries of
// (stage, kind, link) with link = -1 for a same-stage dependency.
int deps(int S, int i, int kind, int out_stage[2], int out_kind[2], int out_link[2]) {
  if (kind == ADAPTRA_OP_F) {
    if (i == 0) return 0;
    out_stage[0] = i - 1; out_kind[0] = ADAPTRA_OP_F; out_link[0] = i - 1;
    return 1;
  }
  if (kind == ADAPTRA_OP_B) {
    if (i == S - 1) {
      out_stage[0] = i; out_kind[0] = ADAPTRA_OP_F; out_link[0] = -1;
    } else {
      out_stage[0] = i + 1; out_kind[0] = ADAPTRA_OP_B; out_link[0] = i;
    }
    return 1;
  }
  out_stage[0] = i; out_kind[0] = ADAPTRA_OP_B; out_link[0] = -1;
  if (i == S - 1) {
    out_stage[1] = i; out_kind[1] = ADAPTRA_OP_F; out_link[1] = -1;
  } else {
    out_stage[1] = i + 1; out_kind[1] = ADAPTRA_OP_B; out_link[1] = i;
  }
  return 2;
}

}  // namespace

extern "C" int adaptra_plan_init(int32_t S, int32_t N, int64_t M, int64_t MF, int32_t* x) {
  if (S < 2 || MF <= 0 || !x) return set_error(ADAPTRA_EINVAL, "plan_init: S >= 2 and M^F > 0 required");
  int64_t x_max = M / MF;                                  // Alg. 1 line max_fwd
  if (N > 0) x_max = std::min<int64_t>(x_max, N);          // R12
  if (x_max < 1) return set_error(ADAPTRA_EINVAL, "plan_init: x_max < 1");
  x[0] = (int32_t)x_max;
  const int64_t d_avg = (x_max - 1) / (S - 1);
  const int64_t r = (x_max - 1) % (S - 1);
  for (int i = 1; i < S; ++i) {
    int64_t d = (i <= r) ? d_avg + 1 : d_avg;
    x[i] = (int32_t)(x[i - 1] - d);
  }
  return ADAPTRA_OK;
}

extern "C" int adaptra_plan_adapt(int32_t S, int32_t N, const int64_t* tF, const int64_t* tB, const int64_t* c,
                                  int32_t* x) {
  if (S < 2 || !tF || !tB || !c || !x) return set_error(ADAPTRA_EINVAL, "plan_adapt: bad arguments");
  for (int i = 0; i < S; ++i)
    if (tF[i] + tB[i] <= 0) return set_error(ADAPTRA_EINVAL, "plan_adapt: non-positive stage time");
  for (int i = 0; i + 1 < S; ++i)
    if (c[i] < 0 || c[i] == ADAPTRA_LINK_DOWN) return set_error(ADAPTRA_EINVAL, "plan_adapt: c must be finite >= 0");
  x[S - 1] = 1;                                             // Alg. 2 line last_stage
  for (int i = S - 2; i >= 0; --i) {
    int64_t need = ceil_div(tF[i] + tB[i] + 2 * c[i], tF[i + 1] + tB[i + 1]);
    int64_t d = std::min<int64_t>((int64_t)N - 2 * S, std::max<int64_t>(need, 2));  // line slackness
    d = std::max<int64_t>(0, d);                                                   // R11
    x[i] = (int32_t)std::min<int64_t>(N, x[i + 1] + d);                           // line fwd_count + R11
  }
  return ADAPTRA_OK;
}

extern "C" int adaptra_eq1_holds(int32_t S, const int64_t* tF, const int64_t* tB, const int64_t* c, const int32_t* x,
                                 uint8_t* ok) {
  if (S < 2 || !tF || !tB || !c || !x || !ok) return set_error(ADAPTRA_EINVAL, "eq1: bad arguments");
  for (int i = 0; i + 1 < S; ++i) {
    int64_t d = x[i] - x[i + 1];
    ok[i] = (tF[i] + tB[i] + 2 * c[i] <= d * (tF[i + 1] + tB[i + 1])) ? 1 : 0;
  }
  return ADAPTRA_OK;
}

extern "C" int adaptra_schedule(int32_t S, int32_t N, const int64_t* tF, const int64_t* tB, const int64_t* tW,
                                const int64_t* c, const int32_t* x, int64_t delta, uint32_t flags,
                                adaptra_op_t* ops, int32_t* n_ops, int64_t* makespan, int64_t* steps_out) {
  if (S < 1 || N < 1 || !tF || !tB || !tW || (S > 1 && !c) || !x || !ops || !n_ops)
    return set_error(ADAPTRA_EINVAL, "schedule: bad arguments");
  if (delta < 1) return set_error(ADAPTRA_EINVAL, "schedule: delta must be >= 1");
  if (!valid_plan(S, N, x)) return set_error(ADAPTRA_EPLAN, "schedule: invalid warm-up plan");
  for (int i = 0; i + 1 < S; ++i)
    if (c[i] < 0 || c[i] == ADAPTRA_LINK_DOWN) return set_error(ADAPTRA_EINVAL, "schedule: c must be finite >= 0");
  const bool merge = flags & ADAPTRA_MERGE_W;
  const bool cap = flags & ADAPTRA_SEL_CAP;
  Dur du(S, tF, tB, tW, merge);
  for (int i = 0; i < S; ++i)
    for (int k = 0; k < 3; ++k)
      if (!(merge && k == ADAPTRA_OP_W) && du.d[k][i] < 1)
        return set_error(ADAPTRA_EINVAL, "schedule: every op duration must be >= 1 tick (R10)");
  std::vector<StageSim> st(S);
  for (int i = 0; i < S; ++i) {
    st[i].x_rem = x[i];
    st[i].x_orig = x[i];
    st[i].avail.reserve(3 * N);
    n_ops[i] = 0;
  }
  for (int j = 1; j <= N; ++j) st[0].avail.push_back({ADAPTRA_OP_F, j, 0});  // A_0 <- [F] x N
  int64_t t = 0, steps = 0, T = 0;
  int64_t pending = N;  // total ops in all A_i
  const int per = 3 * N;
  while (pending > 0) {
    for (int i = 0; i < S; ++i) {
      StageSim& s = st[i];
      if (t < s.end) continue;  // busy (R5)
      int k = select_op(s, t, cap);
      if (k < 0) continue;      // R4
      Avail a = s.avail[k];
      s.avail.erase(s.avail.begin() + k);
      pending -= 1;
      const int64_t end = t + du.d[a.kind][i];
      s.end = end;
      if (a.kind == ADAPTRA_OP_F) s.nF++;
      if (a.kind == ADAPTRA_OP_B) s.nB++;
      if (n_ops[i] >= per) return set_error(ADAPTRA_ENOMEM, "schedule: op overflow");
      ops[(int64_t)i * per + n_ops[i]++] = adaptra_op_t{a.kind, a.mb, t, end};
      T = std::max(T, end);
      if (a.kind == ADAPTRA_OP_F && i != S - 1) {
        st[i + 1].avail.push_back({ADAPTRA_OP_F, a.mb, end + c[i]});         // R1
        pending += 1;
      } else if (a.kind == ADAPTRA_OP_F) {                                    // R2
        s.avail.push_back({ADAPTRA_OP_B, a.mb, end});
        pending += 1;
        if (!merge) {
          s.avail.push_back({ADAPTRA_OP_W, a.mb, end});
          pending += 1;
        }
      } else if (a.kind == ADAPTRA_OP_B && i != 0) {                          // R3
        st[i - 1].avail.push_back({ADAPTRA_OP_B, a.mb, end + c[i - 1]});
        pending += 1;
        if (!merge) {
          st[i - 1].avail.push_back({ADAPTRA_OP_W, a.mb, end + c[i - 1]});  // R8
          pending += 1;
        }
      }
    }
    t += delta;
    steps += 1;
  }
  if (makespan) *makespan = T;
  if (steps_out) *steps_out = steps;
  return ADAPTRA_OK;
}

extern "C" int adaptra_replay(int32_t S, int32_t N, const int64_t* tF, const int64_t* tB, const int64_t* tW,
                              const int64_t* c, const adaptra_op_t* order, const int32_t* n_ops, uint32_t flags,
                              adaptra_op_t* timed, int64_t* makespan) {
  if (S < 1 || N < 1 || !tF || !tB || !tW || (S > 1 && !c) || !order || !n_ops || !timed)
    return set_error(ADAPTRA_EINVAL, "replay: bad arguments");
  const bool merge = flags & ADAPTRA_MERGE_W;
  Dur du(S, tF, tB, tW, merge);
  const int per = 3 * N;
  // done[(stage*3 + kind)*N + (mb-1)] = end time, or -1
  std::vector<int64_t> done((size_t)S * 3 * N, -1);
  std::vector<int> ptr(S, 0);
  std::vector<int64_t> free_t(S, 0);
  int64_t total = 0, n_done = 0, T = 0;
  for (int i = 0; i < S; ++i) {
    if (n_ops[i] < 0 || n_ops[i] > per) return set_error(ADAPTRA_EINVAL, "replay: bad n_ops");
    total += n_ops[i];
  }
  while (n_done < total) {
    bool progress = false;
    for (int i = 0; i < S; ++i) {
      while (ptr[i] < n_ops[i]) {
        const adaptra_op_t& o = order[(int64_t)i * per + ptr[i]];
        if (o.kind < 0 || o.kind > 2 || o.mb < 1 || o.mb > N) return set_error(ADAPTRA_EINVAL, "replay: bad op");
        int ds[2], dk[2], dl[2];
        int nd = deps(S, i, o.kind, ds, dk, dl);
        int64_t ready = free_t[i];
        bool ok = true;
        for (int q = 0; q < nd; ++q) {
          if (merge && dk[q] == ADAPTRA_OP_W) continue;
          int64_t e = done[((size_t)ds[q] * 3 + dk[q]) * N + (o.mb - 1)];
          if (e < 0) {
            ok = false;
            break;
          }
          ready = std::max(ready, e + (dl[q] >= 0 ? c[dl[q]] : 0));
        }
        if (!ok) break;
        const int64_t end = ready + du.d[o.kind][i];
        done[((size_t)i * 3 + o.kind) * N + (o.mb - 1)] = end;
        timed[(int64_t)i * per + ptr[i]] = adaptra_op_t{o.kind, o.mb, ready, end};
        free_t[i] = end;
        T = std::max(T, end);
        ptr[i]++;
        n_done++;
        progress = true;
      }
    }
    if (!progress) return set_error(ADAPTRA_EDEADLOCK, "replay: no stage can progress");
  }
  if (makespan) *makespan = T;
  return ADAPTRA_OK;
}

namespace {
void push_v(adaptra_violation_t* out, int32_t cap, int32_t& n, int32_t code, int32_t stage, int32_t kind, int32_t mb) {
  if (out && n < cap) out[n] = adaptra_violation_t{code, stage, kind, mb};
  n++;
}
}  // namespace

extern "C" int adaptra_validate(int32_t S, int32_t N, const int64_t* tF, const int64_t* tB, const int64_t* tW,
                                const int64_t* c, const adaptra_op_t* ops, const int32_t* n_ops, uint32_t flags,
                                adaptra_violation_t* out, int32_t cap, int32_t* n_viol) {
  if (S < 1 || N < 1 || !tF || !tB || !tW || (S > 1 && !c) || !ops || !n_ops || !n_viol || cap < 0 ||
      (cap > 0 && !out))
    return set_error(ADAPTRA_EINVAL, "validate: bad arguments");
  const bool merge = flags & ADAPTRA_MERGE_W;
  Dur du(S, tF, tB, tW, merge);
  const int per = 3 * N;
  std::vector<int64_t> st((size_t)S * 3 * N, -1), en((size_t)S * 3 * N, -1);
  int32_t v = 0;
  for (int i = 0; i < S; ++i) {
    if (n_ops[i] < 0 || n_ops[i] > per) return set_error(ADAPTRA_EINVAL, "validate: bad n_ops");
    int64_t prev_end = INT64_MIN;
    for (int q = 0; q < n_ops[i]; ++q) {
      const adaptra_op_t& o = ops[(int64_t)i * per + q];
      if (o.kind < 0 || o.kind > 2 || o.mb < 1 || o.mb > N || (merge && o.kind == ADAPTRA_OP_W)) {
        push_v(out, cap, v, ADAPTRA_V_BADOP, i, o.kind, o.mb);
        continue;
      }
      size_t key = ((size_t)i * 3 + o.kind) * N + (o.mb - 1);
      if (st[key] >= 0) push_v(out, cap, v, ADAPTRA_V_DUP, i, o.kind, o.mb);
      st[key] = o.start;
      en[key] = o.end;
      if (o.end - o.start != du.d[o.kind][i]) push_v(out, cap, v, ADAPTRA_V_DURATION, i, o.kind, o.mb);
      if (o.start < prev_end) push_v(out, cap, v, ADAPTRA_V_OVERLAP, i, o.kind, o.mb);
      prev_end = o.end;
    }
    for (int k = 0; k < 3; ++k) {
      if (merge && k == ADAPTRA_OP_W) continue;
      for (int j = 0; j < N; ++j)
        if (st[((size_t)i * 3 + k) * N + j] < 0) push_v(out, cap, v, ADAPTRA_V_MISSING, i, k, j + 1);
    }
  }
  for (int i = 0; i < S; ++i)
    for (int k = 0; k < 3; ++k)
      for (int j = 0; j < N; ++j) {
        int64_t s0 = st[((size_t)i * 3 + k) * N + j];
        if (s0 < 0) continue;
        int ds[2], dk[2], dl[2];
        int nd = deps(S, i, k, ds, dk, dl);
        for (int q = 0; q < nd; ++q) {
          if (merge && dk[q] == ADAPTRA_OP_W) continue;
          int64_t e = en[((size_t)ds[q] * 3 + dk[q]) * N + j];
          if (e < 0) continue;
          if (s0 < e + (dl[q] >= 0 ? c[dl[q]] : 0)) push_v(out, cap, v, ADAPTRA_V_DEP, i, k, j + 1);
        }
      }
  *n_viol = v;
  return ADAPTRA_OK;
}

extern "C" int adaptra_validate_plan(int32_t S, int32_t N, const int32_t* x, adaptra_violation_t* out, int32_t cap,
                                     int32_t* n_viol) {
  if (S < 1 || !x || !n_viol || cap < 0 || (cap > 0 && !out)) return set_error(ADAPTRA_EINVAL, "validate_plan: bad arguments");
  int32_t v = 0;
  for (int i = 0; i + 1 < S; ++i)
    if (x[i] < x[i + 1]) push_v(out, cap, v, ADAPTRA_V_NONMONO, i, -1, 0);
  if (x[S - 1] < 1) push_v(out, cap, v, ADAPTRA_V_X_LAST, S - 1, -1, 0);
  if (x[0] > N) push_v(out, cap, v, ADAPTRA_V_X0_GT_N, 0, -1, 0);
  *n_viol = v;
  return ADAPTRA_OK;
}

extern "C" int adaptra_plan_1f1b(int32_t S, int32_t N, int32_t* x) {
  if (S < 1 || N < 1 || !x) return set_error(ADAPTRA_EINVAL, "plan_1f1b: bad arguments");
  for (int i = 0; i < S; ++i) x[i] = std::min<int32_t>(S - i, N);  // canonical 1F1B warm-ups
  return ADAPTRA_OK;
}

extern "C" int adaptra_clamp_plan(int32_t S, const int32_t* cap, int32_t* x) {
  if (S < 1 || !cap || !x) return set_error(ADAPTRA_EINVAL, "clamp_plan: bad arguments");
  for (int i = 0; i < S; ++i) x[i] = std::min(x[i], cap[i]);       // R26
  for (int i = S - 2; i >= 0; --i) x[i] = std::max(x[i], x[i + 1]);  // Lemma
  return ADAPTRA_OK;
}

extern "C" int64_t adaptra_default_delta(int32_t S, const int64_t* tF, const int64_t* tB, const int64_t* tW,
                                         int32_t ratio) {
  if (S < 1 || !tF || !tB || !tW || ratio < 1) return 1;
  int64_t t_o = 0;
  for (int i = 0; i < S; ++i) t_o = std::max({t_o, tF[i], tB[i], tW[i]});
  return std::max<int64_t>(1, t_o / ratio);  // R10: delta = max(1, floor(t_o / 30))
}

// ---------------------------------------------------------------- planner
// The arm policies (R18, R21, R26) on top of the planning calls above.
struct adaptra_planner {
  int32_t S = 0, N = 0, arm = 0, ratio = 30;
  std::vector<int64_t> tF, tB, tW;           // profile in use
  std::vector<int64_t> ptF, ptB, ptW;        // pending profile (applied at the next re-plan)
  bool pending = false;
  std::vector<int32_t> x, x_init, x_cap;
  std::vector<int64_t> c;                    // latencies the current orders were planned for
  std::vector<adaptra_op_t> ops;             // S * 3N
  std::vector<int32_t> n_ops;
  int64_t makespan = 0, delta = 1, replans = 0;
  bool have = false;

  int plan_for(const int64_t* cv) {
    const uint32_t fl = arm == ADAPTRA_ARM_1F1B ? (ADAPTRA_SEL_CAP | ADAPTRA_MERGE_W) : ADAPTRA_SEL_PAPER;
    int64_t steps = 0;
    return adaptra_schedule(S, N, tF.data(), tB.data(), tW.data(), cv, x.data(), delta, fl, ops.data(), n_ops.data(),
                            &makespan, &steps);
  }
};

extern "C" int adaptra_planner_create(const adaptra_planner_desc_t* d, adaptra_planner_t* out) {
  if (!d || !out || d->S < 2 || d->N < 1 || !d->tF || !d->tB || !d->tW || d->arm < 0 || d->arm > 2)
    return set_error(ADAPTRA_EINVAL, "planner_create: bad arguments");
  auto* p = new adaptra_planner();
  const int S = d->S, N = d->N;
  p->S = S;
  p->N = N;
  p->arm = d->arm;
  p->ratio = d->ratio > 0 ? d->ratio : 30;
  p->tF.assign(d->tF, d->tF + S);
  p->tB.assign(d->tB, d->tB + S);
  p->tW.assign(d->tW, d->tW + S);
  p->x.assign(S, 0);
  p->c.assign(S - 1, 0);
  p->ops.resize((size_t)S * 3 * N);
  p->n_ops.assign(S, 0);
  if (d->x_cap) p->x_cap.assign(d->x_cap, d->x_cap + S);
  p->delta = adaptra_default_delta(S, p->tF.data(), p->tB.data(), p->tW.data(), p->ratio);
  int rc = ADAPTRA_OK;
  if (d->arm == ADAPTRA_ARM_1F1B) {
    rc = adaptra_plan_1f1b(S, N, p->x.data());                              // R21 baseline
  } else if (d->arm == ADAPTRA_ARM_ZB) {
    rc = adaptra_plan_adapt(S, N, p->tF.data(), p->tB.data(), p->c.data(), p->x.data());  // R21: Alg. 2 at c = 0
  } else if (d->x_init) {
    p->x.assign(d->x_init, d->x_init + S);
  } else if (d->mem_per_act > 0) {
    rc = adaptra_plan_init(S, N, d->mem_capacity, d->mem_per_act, p->x.data());  // Alg. 1 (R12)
    if (!rc && !p->x_cap.empty()) rc = adaptra_clamp_plan(S, p->x_cap.data(), p->x.data());
  } else {
    rc = adaptra_plan_adapt(S, N, p->tF.data(), p->tB.data(), p->c.data(), p->x.data());
  }
  if (!rc) rc = p->plan_for(p->c.data());
  if (rc) {
    delete p;
    return rc;
  }
  p->x_init = p->x;
  p->have = true;
  *out = p;
  return ADAPTRA_OK;
}

extern "C" int adaptra_planner_destroy(adaptra_planner_t p) {
  delete p;
  return ADAPTRA_OK;
}

extern "C" int adaptra_planner_set_profile(adaptra_planner_t p, const int64_t* tF, const int64_t* tB,
                                           const int64_t* tW) {
  if (!p || !tF || !tB || !tW) return set_error(ADAPTRA_EINVAL, "planner_set_profile: bad arguments");
  for (int i = 0; i < p->S; ++i)
    if (tF[i] < 1 || tB[i] < 1 || tW[i] < 1) return set_error(ADAPTRA_EINVAL, "planner_set_profile: times >= 1");
  p->ptF.assign(tF, tF + p->S);
  p->ptB.assign(tB, tB + p->S);
  p->ptW.assign(tW, tW + p->S);
  p->pending = true;
  return ADAPTRA_OK;
}

extern "C" int adaptra_planner_step(adaptra_planner_t p, const int64_t* c, adaptra_op_t* ops_out, int32_t* n_ops_out,
                                    int32_t* x_out, int32_t* replanned_out, adaptra_plan_info_t* info) {
  if (!p || !c) return set_error(ADAPTRA_EINVAL, "planner_step: bad arguments");
  const int S = p->S, N = p->N;
  for (int i = 0; i + 1 < S; ++i)
    if (c[i] < 0 || c[i] == ADAPTRA_LINK_DOWN) return set_error(ADAPTRA_EINVAL, "planner_step: c must be finite >= 0");
  int32_t replanned = 0;
  const bool same_c = std::equal(p->c.begin(), p->c.end(), c);
  if (p->arm == ADAPTRA_ARM_ADAPTIVE && !same_c) {
    // R18 at an iteration boundary, with the latest profile (a1)
    if (p->pending) {
      p->tF = p->ptF;
      p->tB = p->ptB;
      p->tW = p->ptW;
      p->pending = false;
      p->delta = adaptra_default_delta(S, p->tF.data(), p->tB.data(), p->tW.data(), p->ratio);
    }
    std::vector<int32_t> xn = p->x;
    bool nominal = true;
    for (int i = 0; i + 1 < S; ++i) nominal = nominal && c[i] == 0;
    if (nominal) {
      xn = p->x_init;                                   // every link nominal: the init plan
    } else {
      std::vector<uint8_t> ok(S - 1);
      int rc = adaptra_eq1_holds(S, p->tF.data(), p->tB.data(), c, p->x.data(), ok.data());
      if (rc) return rc;
      bool all = true;
      for (auto v : ok) all = all && v;
      if (!all) {                                        // Eq. 1 violated: Alg. 2 with the current c
        rc = adaptra_plan_adapt(S, N, p->tF.data(), p->tB.data(), c, xn.data());
        if (!rc && !p->x_cap.empty()) rc = adaptra_clamp_plan(S, p->x_cap.data(), xn.data());  // R26
        if (rc) return rc;
      }
    }
    replanned = xn != p->x;
    p->replans += replanned;
    p->x = xn;
    p->c.assign(c, c + S - 1);
    int rc = p->plan_for(p->c.data());
    if (rc) return rc;
  }
  if (ops_out) std::copy(p->ops.begin(), p->ops.end(), ops_out);
  if (n_ops_out) std::copy(p->n_ops.begin(), p->n_ops.end(), n_ops_out);
  if (x_out) std::copy(p->x.begin(), p->x.end(), x_out);
  if (replanned_out) *replanned_out = replanned;
  if (info) {
    info->makespan = p->makespan;
    info->delta = p->delta;
    info->replans = p->replans;
    for (int i = 0; i < S && i < ADAPTRA_MAX_STAGES; ++i) {
      info->tF[i] = p->tF[i];
      info->tB[i] = p->tB[i];
      info->tW[i] = p->tW[i];
    }
  }
  return ADAPTRA_OK;
}
