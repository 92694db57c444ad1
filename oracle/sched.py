"""CPU oracle for Adaptra's scheduling method (arXiv 2504.19232).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this module.
The product path (``paper_2504_19232_b200``) never imports it and shares no
code with it.

Everything here is plain Python on integers (time in int ticks; the product
side uses int64 nanoseconds).  Each function follows the paper's pseudocode in
its order and notation.  Citations are ``P:<line>`` into PAPER.md (main.tex
copy) and ``R<k>`` into the ambiguity register in DESIGN.md §3.

Pins (tests/test_oracle_sched.py): paper-printed makespans 390/400/440 ms and
S_0's B_1 at 110 ms, the per-stage op order of the ideal
ZB figure, the 1F1B closed form T=(N+S-1)(tF+tB+tW) and bubble (S-1)/(N+S-1),
the ZB closed form (S-1)tF+N(tF+tB+tW), the Lemma x_i >= x_{i+1},
hand traces of Alg. 1/2, Eq. 1 boundaries, Theorem 1 regimes, dependency
validity of every emitted schedule, and brute-force optimality on tiny cases.
The checkers are pinned negatively: a mutated copy of the ideal schedule is
flagged with each violation class (dup, missing, duration, overlap, dep of
F / B / W, badop), and non-monotone / out-of-range plans are rejected; the
R26 clamp and the R18 policy are pinned by hand traces; P2's interior and
utilisation bubbles (0.0886 / 0.182) from the printed 440 ms; P11 against an
exact branch-and-bound optimum at the paper's smallest setting (S=3, N=6),
itself cross-checked against exhaustive search on S=2.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

F, B, W = "F", "B", "W"
# Execution priority after warm-up: B > F > W  (Alg. SelectOp)
PRI = {B: 3, F: 2, W: 1}

MODE_PAPER = "paper"  # literal greedy SelectOp (R7, default)
MODE_CAP = "cap"      # F eligible only while (#F started - #B started) < x_i (R7; 1F1B / ZB-H1)

INF = float("inf")


class PlanError(ValueError):
    pass


class DeadlockError(RuntimeError):
    pass


# ---------------------------------------------------------------------------
# §4.2 Orchestrating warm-up forwards
# ---------------------------------------------------------------------------

def get_init_warmup_fwds(S: int, M: int, MF: int, N: int | None = None) -> list[int]:
    """Alg. 1 "Initial Planning".

    x_max = floor(M / M^F) (line max_fwd); x_0 = x_max; Delta_avg =
    floor((x_max-1)/(S-1)); r = (x_max-1) mod (S-1); for i = 1..S-1:
    Delta_{i-1} = Delta_avg + 1 if i <= r else Delta_avg; x_i = x_{i-1} - Delta_{i-1}.
    R12: when N is given, x_max is clamped to N (more warm-up forwards than
    microbatches do not exist).
    """
    if S < 2:
        raise PlanError("S must be >= 2")
    x_max = M // MF
    if N is not None:
        x_max = min(x_max, N)
    if x_max < 1:
        raise PlanError("x_max < 1: not even one activation fits")
    x = [0] * S
    x[0] = x_max
    d_avg = (x_max - 1) // (S - 1)
    r = (x_max - 1) % (S - 1)
    for i in range(1, S):
        d = d_avg + 1 if i <= r else d_avg
        x[i] = x[i - 1] - d
    return x


def ceil_div(a: int, b: int) -> int:
    return -((-a) // b)


def get_adapted_warmup_fwds(S: int, N: int, tF, tB, c) -> list[int]:
    """Alg. 2 "Dynamic Adaptation".

    x_{S-1} = 1; for i = S-2..0:
      Delta_i = min(N-2S, max(ceil((tF_i + tB_i + 2c_i) / (tF_{i+1} + tB_{i+1})), 2))
      x_i = x_{i+1} + Delta_i
    R11: Delta_i is floored at 0 (N-2S < 0 when N < 2S) and x_i is capped at N.
    """
    if S < 2:
        raise PlanError("S must be >= 2")
    x = [0] * S
    x[S - 1] = 1
    for i in range(S - 2, -1, -1):
        need = ceil_div(tF[i] + tB[i] + 2 * c[i], tF[i + 1] + tB[i + 1])
        d = min(N - 2 * S, max(need, 2))
        d = max(0, d)                      # R11
        x[i] = min(N, x[i + 1] + d)        # R11
    return x


def eq1_holds(tF, tB, c, x) -> list[bool]:
    """Eq. 1 absorption condition per link i:
    tF_i + tB_i + 2 c_i <= Delta_i (tF_{i+1} + tB_{i+1}), Delta_i = x_i - x_{i+1}."""
    S = len(x)
    out = []
    for i in range(S - 1):
        d = x[i] - x[i + 1]
        out.append(tF[i] + tB[i] + 2 * c[i] <= d * (tF[i + 1] + tB[i + 1]))
    return out


def slackness(x) -> list[int]:
    """Delta_i = x_i - x_{i+1}."""
    return [x[i] - x[i + 1] for i in range(len(x) - 1)]


def plan_violations(N: int, x) -> list[tuple]:
    """Lemma: x non-increasing; plus x_{S-1} >= 1 (Alg. 1/2 set
    the last stage's count to 1) and x_0 <= N (R11: there
    are only N forwards).  Returns (code, index) tuples; codes "nonmono" (at
    link i), "x_last", "x0_gt_N"."""
    v = []
    for i in range(len(x) - 1):
        if x[i] < x[i + 1]:
            v.append(("nonmono", i))
    if x[-1] < 1:
        v.append(("x_last", len(x) - 1))
    if x[0] > N:
        v.append(("x0_gt_N", 0))
    return v


def validate_plan(N: int, x) -> list[str]:
    """plan_violations as readable strings ([] = valid plan)."""
    return [f"{code} at {i}" for code, i in plan_violations(N, x)]


# ---------------------------------------------------------------------------
# §4.3 / Appendix: SelectOp (Alg. 3) and Schedule (Alg. 4)
# ---------------------------------------------------------------------------

@dataclass
class Op:
    kind: str
    mb: int          # 1-based microbatch index, as in the paper's figures
    start: int = 0
    end: int = 0


@dataclass
class _StageState:
    x_rem: int                  # remaining warm-up forwards (x_i, decremented by SelectOp)
    x_orig: int
    avail: list = field(default_factory=list)  # A_i: list of (kind, mb, ready)
    end: int = 0                # end time of the op currently executing (busy <=> t < end, R5)
    nF: int = 0
    nB: int = 0


def select_op(st: _StageState, t: int, mode: str):
    """Alg. 3 SelectOp(i, A_i, x_i).

    Only operators whose ready time is <= t are in A_i at step t (R5).
    Returns the popped (kind, mb) or None (R4: the stage idles this step).
    """
    cand = [a for a in st.avail if a[2] <= t]
    if not cand:                                   # A_i = {} -> None
        return None
    # Warm-up phase: do x_i forwards at first.
    if st.x_rem > 0:
        fs = [a for a in cand if a[0] == F]
        if fs:
            st.x_rem -= 1
            a = min(fs, key=lambda a: a[1])        # R6: lowest microbatch
            st.avail.remove(a)
            return a
        return None
    # Execution priority after warm-up: B > F > W.
    if mode == MODE_CAP:
        # R7 CAP reading: F eligible only while in-flight forwards < x_i.
        if st.nF - st.nB >= st.x_orig:
            cand = [a for a in cand if a[0] != F]
            if not cand:
                return None
    best = max(PRI[a[0]] for a in cand)
    a = min((a for a in cand if PRI[a[0]] == best), key=lambda a: a[1])  # R6
    st.avail.remove(a)
    return a


def schedule(S, N, tF, tB, tW, c, x, delta, mode=MODE_PAPER, merge_w=False):
    """Alg. 4 Schedule(S, N, {tF},{tB},{tW},{x},{c}, delta).

    Returns (X, T, steps): X[i] = list of Op in execution order on stage i;
    T = max end time (R9); steps = number of delta iterations (R9).

    Readings: successor ready = completion + c (R1); the last stage's F makes
    its own B and W available at completion (R2); "s != 0" read as i != 0
    (R3); W_{i-1} appended with B_{i-1} at the same ready time (R8);
    merge_w (1F1B) folds tW into B and creates no W (R10).
    """
    if delta < 1:
        raise PlanError("delta must be >= 1 tick")
    if validate_plan(N, x):
        raise PlanError("invalid warm-up plan: " + ";".join(validate_plan(N, x)))
    dur = {}
    for i in range(S):
        dur[(i, F)] = tF[i]
        dur[(i, B)] = tB[i] + (tW[i] if merge_w else 0)
        dur[(i, W)] = tW[i]
    st = [_StageState(x_rem=x[i], x_orig=x[i]) for i in range(S)]
    st[0].avail = [(F, j, 0) for j in range(1, N + 1)]      # A_0 <- [F] x N
    X = [[] for _ in range(S)]
    t = 0
    steps = 0
    while any(s.avail for s in st):
        for i in range(S):
            s = st[i]
            if t < s.end:                                  # i.busy()
                continue
            o = select_op(s, t, mode)
            if o is None:
                continue
            kind, mb, _ = o
            end = t + dur[(i, kind)]
            s.end = end
            if kind == F:
                s.nF += 1
            elif kind == B:
                s.nB += 1
            X[i].append(Op(kind, mb, t, end))
            # Add dependent operators after execution.
            if kind == F and i != S - 1:
                st[i + 1].avail.append((F, mb, end + c[i]))
            elif kind == F and i == S - 1:                 # R2
                s.avail.append((B, mb, end))
                if not merge_w:
                    s.avail.append((W, mb, end))
            elif kind == B and i != 0:                     # R3
                st[i - 1].avail.append((B, mb, end + c[i - 1]))
                if not merge_w:
                    st[i - 1].avail.append((W, mb, end + c[i - 1]))
        t += delta
        steps += 1
    T = max(op.end for ops in X for op in ops)
    return X, T, steps


# ---------------------------------------------------------------------------
# Fixed-order replay (event driven, exact; no delta)  -- dependency rules A1
# ---------------------------------------------------------------------------

def _deps(S, i, kind, mb):
    """Dependencies of op (i, kind, mb) per P:1743-1753 plus R8 (W after own B).
    Returns list of ((stage, kind, mb), link latency index or None)."""
    if kind == F:
        return [((i - 1, F, mb), i - 1)] if i > 0 else []
    if kind == B:
        if i == S - 1:
            return [((i, F, mb), None)]
        return [((i + 1, B, mb), i)]
    # W: same availability as B and after its own B (R8)
    d = [((i, B, mb), None)]
    if i == S - 1:
        d.append(((i, F, mb), None))
    else:
        d.append(((i + 1, B, mb), i))
    return d


def replay(S, N, tF, tB, tW, c, order, merge_w=False):
    """Execute per-stage op orders as early as dependencies and the stage allow.

    order[i] = list of (kind, mb).  Returns timed X (list of Op per stage) and T.
    Raises DeadlockError when no stage can progress.
    """
    dur = {}
    for i in range(S):
        dur[(i, F)] = tF[i]
        dur[(i, B)] = tB[i] + (tW[i] if merge_w else 0)
        dur[(i, W)] = tW[i]
    done = {}
    ptr = [0] * S
    free = [0] * S
    X = [[] for _ in range(S)]
    total = sum(len(o) for o in order)
    n_done = 0
    while n_done < total:
        progress = False
        for i in range(S):
            while ptr[i] < len(order[i]):
                kind, mb = order[i][ptr[i]]
                ready = free[i]
                ok = True
                for (dep, link) in _deps(S, i, kind, mb):
                    if merge_w and dep[1] == W:
                        continue
                    if dep not in done:
                        ok = False
                        break
                    ready = max(ready, done[dep] + (c[link] if link is not None else 0))
                if not ok:
                    break
                end = ready + dur[(i, kind)]
                done[(i, kind, mb)] = end
                X[i].append(Op(kind, mb, ready, end))
                free[i] = end
                ptr[i] += 1
                n_done += 1
                progress = True
        if not progress:
            raise DeadlockError("replay cannot progress")
    T = max(op.end for ops in X for op in ops)
    return X, T


def order_of(X):
    return [[(op.kind, op.mb) for op in ops] for ops in X]


# ---------------------------------------------------------------------------
# Validation and metrics
# ---------------------------------------------------------------------------

def violations(S, N, tF, tB, tW, c, X, merge_w=False) -> list[tuple]:
    """Check a timed schedule against the problem's constraints and return
    every violation as (code, stage, kind, mb):

      "badop"    kind not F/B/W, mb outside 1..N, or a W op in a merged
                 (1F1B) schedule, which has none (R10);
      "dup"      the op appears twice on its stage;
      "missing"  an op of the stage's 3N (2N merged) is absent;
      "duration" end - start != the stage's op time (B + W merged, R10);
      "overlap"  the op starts before the previous op on its stage ended
                 (one op at a time per stage, P:2754 busy());
      "dep"      the op starts before a dependency's end + link latency:
                 F after the upstream F + c (R1); B after the
                 downstream B + c, or after its own F on the last stage
                 (R2); W after its own B and the B that makes
                 it available (R8).
    A valid schedule returns []."""
    v = []
    kinds = (F, B) if merge_w else (F, B, W)
    end = {}
    for i in range(S):
        seen = set()
        prev_end = None
        for op in X[i]:
            if op.kind not in kinds or not 1 <= op.mb <= N:
                v.append(("badop", i, op.kind, op.mb))
                continue
            key = (op.kind, op.mb)
            if key in seen:
                v.append(("dup", i, op.kind, op.mb))
            seen.add(key)
            want = {F: tF[i], B: tB[i] + (tW[i] if merge_w else 0), W: tW[i]}[op.kind]
            if op.end - op.start != want:
                v.append(("duration", i, op.kind, op.mb))
            if prev_end is not None and op.start < prev_end:
                v.append(("overlap", i, op.kind, op.mb))
            prev_end = op.end
            end[(i, op.kind, op.mb)] = (op.start, op.end)
        for k in kinds:
            for j in range(1, N + 1):
                if (k, j) not in seen:
                    v.append(("missing", i, k, j))
    for (i, k, j), (s, _e) in end.items():
        for (dep, link) in _deps(S, i, k, j):
            if merge_w and dep[1] == W:
                continue
            if dep not in end:
                continue
            need = end[dep][1] + (c[link] if link is not None else 0)
            if s < need:
                v.append(("dep", i, k, j))
    return v


def validate(S, N, tF, tB, tW, c, X, merge_w=False) -> list[str]:
    """violations() as readable strings ([] = valid schedule)."""
    return [f"{code} {k}{j} on stage {i}" for code, i, k, j in violations(S, N, tF, tB, tW, c, X, merge_w)]


def metrics(S, X, T=None) -> dict:
    """Bubble rates (R15), peak in-flight, measured warm-up counts."""
    if T is None:
        T = max(op.end for ops in X for op in ops)
    busy = [sum(op.end - op.start for op in ops) for ops in X]
    span = [(ops[-1].end - ops[0].start) if ops else 0 for ops in X]
    util = 1.0 - sum(busy) / (S * T)
    interior = (sum(sp - b for sp, b in zip(span, busy)) / sum(span)) if sum(span) else 0.0
    peak_fb, peak_fw, warm = [], [], []
    for ops in X:
        nf = nb = nw = 0
        pfb = pfw = 0
        m = None
        for op in ops:
            if op.kind == F:
                nf += 1
            elif op.kind == B:
                nb += 1
                if m is None:
                    m = nf
            else:
                nw += 1
            pfb = max(pfb, nf - nb)
            pfw = max(pfw, nf - nw)
        peak_fb.append(pfb)
        peak_fw.append(pfw)
        warm.append(m if m is not None else nf)
    return {"T": T, "busy": busy, "util_bubble": util, "interior_bubble": interior,
            "peak_inflight": peak_fb, "peak_stash": peak_fw, "warmup": warm}


def lower_bound_c(S, N, tF, tB, tW, c) -> int:
    """LB_c = sum_{i<S-1}(tF_i + c_i) + N (tF+tB+tW)_{S-1}: the last stage cannot
    start before the first microbatch reaches it and then has 3N ops to run."""
    return sum(tF[i] + c[i] for i in range(S - 1)) + N * (tF[S - 1] + tB[S - 1] + tW[S - 1])


def default_delta(tF, tB, tW, ratio=30) -> int:
    """R10: delta = max(1, floor(t_o / 30)), t_o = max op time."""
    t_o = max(max(tF), max(tB), max(tW))
    return max(1, t_o // ratio)


# ---------------------------------------------------------------------------
# Baselines (R21) and the adaptive policy (R18)
# ---------------------------------------------------------------------------

def plan_1f1b(S, N):
    return [min(S - i, N) for i in range(S)]


def schedule_1f1b(S, N, tF, tB, tW, delta):
    """1F1B = Schedule(CAP, MERGE_W, x_i = min(S-i, N), c=0) (A13)."""
    return schedule(S, N, tF, tB, tW, [0] * (S - 1), plan_1f1b(S, N), delta,
                    mode=MODE_CAP, merge_w=True)


def schedule_zb(S, N, tF, tB, tW, delta):
    """ZB = Schedule(PAPER, x = Alg.2 at c=0) (A14, R21)."""
    x = get_adapted_warmup_fwds(S, N, tF, tB, [0] * (S - 1))
    return schedule(S, N, tF, tB, tW, [0] * (S - 1), x, delta, mode=MODE_PAPER)


def adaptive_plan(S, N, tF, tB, c, x_cur, x_init, c_nominal=None):
    """R18 re-plan rule at an iteration boundary.

    Returns (x_new, replanned).  If Eq. 1 fails on some link under the current
    plan -> Alg. 2 with the current c.  If every link is back to nominal ->
    revert to the init plan.  Otherwise keep the current plan.
    """
    if c_nominal is None:
        c_nominal = [0] * (S - 1)
    if all(ci <= cn for ci, cn in zip(c, c_nominal)):
        return list(x_init), list(x_init) != list(x_cur)
    if not all(eq1_holds(tF, tB, c, x_cur)):
        x = get_adapted_warmup_fwds(S, N, tF, tB, c)
        return x, x != list(x_cur)
    return list(x_cur), False


def clamp_plan(x, cap):
    """R26: without host activation offload (N4) the device stash caps the
    warm-up counts: x_i <- min(x_i, cap_i), then the Lemma is
    restored from the last stage upwards, x_i <- max(x_i, x_{i+1})."""
    out = [min(v, c) for v, c in zip(x, cap)]
    for i in range(len(out) - 2, -1, -1):
        out[i] = max(out[i], out[i + 1])
    return out


def adaptive_step(S, N, tF, tB, tW, c, x_prev, x_init, x_cap=None, ratio=30):
    """One iteration boundary of the adaptive arm (R18): every link nominal ->
    the init plan; Eq. 1 violated on some link under the
    current plan -> Alg. 2 with the current c, clamped by R26;
    otherwise the current plan is kept.  Returns (x, per-stage (kind, mb)
    order of Schedule() under c with delta = t_o / ratio, R10)."""
    if all(v == 0 for v in c):
        x = list(x_init)
    elif not all(eq1_holds(tF, tB, c, x_prev)):
        xa = get_adapted_warmup_fwds(S, N, tF, tB, c)
        x = clamp_plan(xa, x_cap) if x_cap else xa
    else:
        x = list(x_prev)
    X, _, _ = schedule(S, N, tF, tB, tW, c, x, default_delta(tF, tB, tW, ratio))
    return x, order_of(X)


def adaptive_orders(S, N, tF, tB, tW, cs_seq, x_init, x_cap=None, ratio=30):
    """The adaptive arm over a sequence of per-iteration latency vectors
    (R18): returns [(x, per-stage (kind, mb) order)] for every iteration."""
    x = list(x_init)
    out = []
    for c in cs_seq:
        x, order = adaptive_step(S, N, tF, tB, tW, c, x, x_init, x_cap, ratio)
        out.append((list(x), order))
    return out


# ---------------------------------------------------------------------------
# Brute force optimum on tiny instances (stand-in for the paper's MILP, A12)
# ---------------------------------------------------------------------------

def brute_force_optimum(S, N, tF, tB, tW, c):
    """Minimum makespan over all dependency-respecting per-stage orders, by
    exhaustive search of list schedules (each stage picks its next op among
    all remaining ops, then replay timing).  Tiny inputs only."""
    best = [INF]
    ops_all = [[(k, j) for j in range(1, N + 1) for k in (F, B, W)] for _ in range(S)]

    def rec(orders, remaining):
        if all(not r for r in remaining):
            try:
                _, T = replay(S, N, tF, tB, tW, c, orders)
            except DeadlockError:
                return
            best[0] = min(best[0], T)
            return
        # extend the first stage that still has ops (enumerate its full order)
        i = next(k for k, r in enumerate(remaining) if r)
        placed = set(orders[i])
        for op in list(remaining[i]):
            k, j = op
            if k == B and (F, j) not in placed:
                continue
            if k == W and (B, j) not in placed:
                continue
            if k == F and j > 1 and (F, j - 1) not in placed:
                continue          # forwards in microbatch order (WLOG: identical ops)
            orders[i].append(op)
            remaining[i].remove(op)
            rec(orders, remaining)
            remaining[i].append(op)
            orders[i].pop()

    rec([[] for _ in range(S)], [list(o) for o in ops_all])
    return best[0]


def exact_optimum(S, N, tF, tB, tW, c, ub=None):
    """Minimum makespan over ALL feasible schedules (no restriction on the
    per-stage orders), by branch and bound over active schedules.

    Each stage is a machine that runs one op at a time; an op may start once
    every dependency of `_deps` has ended plus its link latency (P:1743-1753,
    R1, R8).  Some optimal schedule is active (no op can start earlier without
    delaying another), and Giffler-Thompson generation enumerates every active
    schedule: take the schedulable op o* with the earliest possible
    completion e*, on stage m*; branch on every schedulable op of m* that can
    start before e*.  Pruning: a stage cannot finish before its free time
    plus its remaining work, and (one-machine relaxation) not before the
    earliest head of its unscheduled ops + their work + the shortest tail
    (longest dependency chain that must follow an op).  Symmetry:
    microbatches are identical, so among candidates of the same stage and
    kind whose microbatches have identical histories only one is tried.
    Tiny inputs only (S <= 4, N <= 8)."""
    kinds = (F, B, W)
    dur = {(i, F): tF[i] for i in range(S)}
    dur.update({(i, B): tB[i] for i in range(S)})
    dur.update({(i, W): tW[i] for i in range(S)})
    # topological order of one microbatch's ops: F down the stages, B back up, W
    topo = [(i, F) for i in range(S)] + [(i, B) for i in range(S - 1, -1, -1)] + [(i, W) for i in range(S)]
    allops = [(i, k, j) for j in range(1, N + 1) for (i, k) in topo]
    deps = {op: _deps(S, *op) for op in allops}
    succ = {op: [] for op in allops}
    for op in allops:
        for dep, link in deps[op]:
            succ[dep].append((op, c[link] if link is not None else 0))
    tail = {}
    for op in reversed(allops):
        tail[op] = max((lag + dur[(s[0], s[1])] + tail[s] for s, lag in succ[op]), default=0)
    end = {}
    free = [0] * S
    rem = [N * (tF[i] + tB[i] + tW[i]) for i in range(S)]
    best = [INF if ub is None else ub + 1]

    def history(j):
        return tuple(end.get((i, k, j), -1) for i in range(S) for k in kinds)

    def jackson(jobs):
        """Preemptive one-machine bound: jobs (release, duration, tail); run
        the released job with the largest tail, preempting on arrivals;
        returns max(completion + tail) (a lower bound on that machine)."""
        jobs = sorted(jobs)
        t, k, lb = 0, 0, 0
        ready = []                      # [-tail, remaining]
        while k < len(jobs) or ready:
            if not ready and t < jobs[k][0]:
                t = jobs[k][0]
            while k < len(jobs) and jobs[k][0] <= t:
                ready.append([-jobs[k][2], jobs[k][1]])
                k += 1
            ready.sort()
            nxt = jobs[k][0] if k < len(jobs) else INF
            run = min(ready[0][1], nxt - t)
            t += run
            ready[0][1] -= run
            if ready[0][1] == 0:
                lb = max(lb, t - ready[0][0])
                ready.pop(0)
        return lb

    def lower_bound():
        head = {}
        jobs = [[] for _ in range(S)]
        for op in allops:
            if op in end:
                continue
            h = free[op[0]]
            for dep, link in deps[op]:
                fin = end[dep] if dep in end else head[dep] + dur[(dep[0], dep[1])]
                h = max(h, fin + (c[link] if link is not None else 0))
            head[op] = h
            jobs[op[0]].append((h, dur[(op[0], op[1])], tail[op]))
        return max(max(free), max(jackson(js) for js in jobs))

    seen_states = set()

    def rec(n_left):
        if n_left == 0:
            best[0] = min(best[0], max(free))
            return
        if lower_bound() >= best[0]:
            return
        # the same partial schedule up to a relabelling of the (identical)
        # microbatches, reached by another branch order
        key = (tuple(free), tuple(sorted(history(j) for j in range(1, N + 1))))
        if key in seen_states:
            return
        seen_states.add(key)
        cand = []
        for op in allops:
            if op in end:
                continue
            r = 0
            ok = True
            for dep, link in deps[op]:
                if dep not in end:
                    ok = False
                    break
                r = max(r, end[dep] + (c[link] if link is not None else 0))
            if ok:
                es = max(r, free[op[0]])
                cand.append((es + dur[(op[0], op[1])], es, op))
        e_star, _, o_star = min(cand)
        m = o_star[0]
        seen = set()
        for e, es, op in sorted(cand):
            if op[0] != m or es >= e_star:
                continue
            sig = (op[1], es, history(op[2]))
            if sig in seen:
                continue
            seen.add(sig)
            i, k, _ = op
            old = free[i]
            end[op] = e
            free[i] = e
            rem[i] -= dur[(i, k)]
            rec(n_left - 1)
            rem[i] += dur[(i, k)]
            free[i] = old
            del end[op]

    rec(len(allops))
    return best[0]
