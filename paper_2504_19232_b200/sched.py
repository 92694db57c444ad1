"""Python binding of the host scheduling core (csrc/sched/sched.cpp).

Marshalling only; the planning and simulation run in libadaptra.so.
Ops are returned as per-stage lists of (kind, mb, start, end) with kind in
"F"/"B"/"W" and 1-based microbatches.
"""
from __future__ import annotations

import ctypes as C

from . import _lib as L

KIND = {L.OP_F: "F", L.OP_B: "B", L.OP_W: "W"}
KIND_ID = {"F": L.OP_F, "B": L.OP_B, "W": L.OP_W}


def _arr(t, vals):
    return (t * len(vals))(*vals)


def plan_init(S, N, mem, mem_per_act):
    x = (C.c_int32 * S)()
    L.check(L.lib().adaptra_plan_init(S, N, mem, mem_per_act, x))
    return list(x)


def plan_adapt(S, N, tF, tB, c):
    x = (C.c_int32 * S)()
    L.check(L.lib().adaptra_plan_adapt(S, N, _arr(C.c_int64, tF), _arr(C.c_int64, tB),
                                       _arr(C.c_int64, list(c) or [0]), x))
    return list(x)


def eq1_holds(tF, tB, c, x):
    S = len(x)
    ok = (C.c_uint8 * max(1, S - 1))()
    L.check(L.lib().adaptra_eq1_holds(S, _arr(C.c_int64, tF), _arr(C.c_int64, tB),
                                      _arr(C.c_int64, list(c) or [0]), _arr(C.c_int32, x), ok))
    return [bool(v) for v in ok[:S - 1]]


def _flags(mode, merge_w):
    return (L.SEL_CAP if mode == "cap" else L.SEL_PAPER) | (L.MERGE_W if merge_w else 0)


def schedule(S, N, tF, tB, tW, c, x, delta, mode="paper", merge_w=False):
    """Alg. 4 Schedule.  Returns (X, T, steps), X[i] = [(kind, mb, start, end)]."""
    per = 3 * N
    ops = (L.Op * (S * per))()
    n = (C.c_int32 * S)()
    T = C.c_int64()
    steps = C.c_int64()
    L.check(L.lib().adaptra_schedule(S, N, _arr(C.c_int64, tF), _arr(C.c_int64, tB), _arr(C.c_int64, tW),
                                      _arr(C.c_int64, list(c) or [0]), _arr(C.c_int32, x), delta,
                                      _flags(mode, merge_w), ops, n, C.byref(T), C.byref(steps)))
    X = [[(KIND[ops[i * per + q].kind], ops[i * per + q].mb, ops[i * per + q].start, ops[i * per + q].end)
          for q in range(n[i])] for i in range(S)]
    return X, T.value, steps.value


def _pack(S, N, order):
    per = 3 * N
    arr = (L.Op * (S * per))()
    n = (C.c_int32 * S)()
    for i in range(S):
        n[i] = len(order[i])
        for q, o in enumerate(order[i]):
            arr[i * per + q].kind = KIND_ID[o[0]]
            arr[i * per + q].mb = o[1]
            if len(o) >= 4:
                arr[i * per + q].start = o[2]
                arr[i * per + q].end = o[3]
    return arr, n


def replay(S, N, tF, tB, tW, c, order, merge_w=False):
    per = 3 * N
    arr, n = _pack(S, N, order)
    out = (L.Op * (S * per))()
    T = C.c_int64()
    L.check(L.lib().adaptra_replay(S, N, _arr(C.c_int64, tF), _arr(C.c_int64, tB), _arr(C.c_int64, tW),
                                   _arr(C.c_int64, list(c) or [0]), arr, n, _flags("paper", merge_w), out,
                                   C.byref(T)))
    X = [[(KIND[out[i * per + q].kind], out[i * per + q].mb, out[i * per + q].start, out[i * per + q].end)
          for q in range(n[i])] for i in range(S)]
    return X, T.value


def validate(S, N, tF, tB, tW, c, X, merge_w=False, cap=4096):
    """adaptra_validate: [(code, stage, kind, mb)] with the codes of
    L.V_CODES ("dep", "overlap", ...) and kinds "F"/"B"/"W"; [] = valid."""
    arr, n = _pack(S, N, X)
    out = (L.Violation * cap)()
    v = C.c_int32()
    L.check(L.lib().adaptra_validate(S, N, _arr(C.c_int64, tF), _arr(C.c_int64, tB), _arr(C.c_int64, tW),
                                     _arr(C.c_int64, list(c) or [0]), arr, n, _flags("paper", merge_w), out, cap,
                                     C.byref(v)))
    return [(L.V_CODES[o.code], o.stage, KIND.get(o.kind, o.kind), o.mb) for o in out[:min(cap, v.value)]]


def validate_plan(S, N, x, cap=256):
    out = (L.Violation * cap)()
    v = C.c_int32()
    L.check(L.lib().adaptra_validate_plan(S, N, _arr(C.c_int32, x), out, cap, C.byref(v)))
    return [(L.V_CODES[o.code], o.stage) for o in out[:min(cap, v.value)]]


def plan_1f1b(S, N):
    x = (C.c_int32 * S)()
    L.check(L.lib().adaptra_plan_1f1b(S, N, x))
    return list(x)


def clamp_plan(x, cap):
    xs = _arr(C.c_int32, x)
    L.check(L.lib().adaptra_clamp_plan(len(x), _arr(C.c_int32, cap), xs))
    return list(xs)


def default_delta(tF, tB, tW, ratio=30):
    return L.lib().adaptra_default_delta(len(tF), _arr(C.c_int64, tF), _arr(C.c_int64, tB), _arr(C.c_int64, tW),
                                         ratio)


def nccl_post_plan(orders, merge_w=False, buffered=0):
    """adaptra_nccl_post_plan (R39): per stage, for each op the index of the
    group that posts its receive (-1: no receive); `buffered` = messages a
    link holds without a posted receive."""
    S = len(orders)
    flat = [o for ops in orders for o in ops]
    arr = (L.Op * max(1, len(flat)))()
    for q, (k, mb) in enumerate(flat):
        arr[q].kind = KIND_ID[k]
        arr[q].mb = mb
    post = (C.c_int32 * max(1, len(flat)))()
    L.check(L.lib().adaptra_nccl_post_plan(S, arr, _arr(C.c_int32, [len(o) for o in orders]),
                                          _flags("paper", merge_w), int(buffered), post))
    out, base = [], 0
    for ops in orders:
        out.append(list(post[base:base + len(ops)]))
        base += len(ops)
    return out


class Planner:
    """adaptra_planner_*: one schedule arm (1F1B / ZB / adaptive, R18/R21/R26)."""

    ARMS = {"1f1b": L.ARM_1F1B, "zb": L.ARM_ZB, "adaptive": L.ARM_ADAPTIVE}

    def __init__(self, arm, S, N, tF, tB, tW, *, x_init=None, x_cap=None, mem=None, ratio=30):
        d = L.PlannerDesc()
        d.S, d.N, d.arm, d.ratio = S, N, self.ARMS[arm], ratio
        self._keep = [_arr(C.c_int64, tF), _arr(C.c_int64, tB), _arr(C.c_int64, tW)]
        d.tF, d.tB, d.tW = self._keep
        if x_init is not None:
            self._keep.append(_arr(C.c_int32, x_init))
            d.x_init = self._keep[-1]
        if x_cap is not None:
            self._keep.append(_arr(C.c_int32, x_cap))
            d.x_cap = self._keep[-1]
        if mem is not None:
            d.mem_capacity, d.mem_per_act = mem
        self.S, self.N, self.arm = S, N, arm
        self.h = C.c_void_p()
        L.check(L.lib().adaptra_planner_create(C.byref(d), C.byref(self.h)))
        self.info = L.PlanInfo()

    def set_profile(self, tF, tB, tW):
        L.check(L.lib().adaptra_planner_set_profile(self.h, _arr(C.c_int64, tF), _arr(C.c_int64, tB),
                                                    _arr(C.c_int64, tW)))

    def step(self, c):
        """Returns (orders, x, replanned): orders[i] = [(kind, mb), ...]."""
        S, per = self.S, 3 * self.N
        ops = (L.Op * (S * per))()
        n = (C.c_int32 * S)()
        x = (C.c_int32 * S)()
        r = C.c_int32()
        L.check(L.lib().adaptra_planner_step(self.h, _arr(C.c_int64, list(c) or [0]), ops, n, x, C.byref(r),
                                             C.byref(self.info)))
        orders = [[(KIND[ops[i * per + q].kind], ops[i * per + q].mb) for q in range(n[i])] for i in range(S)]
        return orders, list(x), bool(r.value)

    @property
    def profile(self):
        S = self.S
        return list(self.info.tF[:S]), list(self.info.tB[:S]), list(self.info.tW[:S])

    def close(self):
        if self.h:
            L.lib().adaptra_planner_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def order_of(X):
    return [[(o[0], o[1]) for o in ops] for ops in X]
