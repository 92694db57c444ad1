"""N4 host stash offload: the executor's per-iteration offload
plan (adaptra_offload_plan, host code) replayed by a simulator of the device
and host slot pools on schedules of every arm: every op finds its
microbatch's data in the device slot the plan gives it, no slot is shared by
two live microbatches, only complete slots (B done) move to the host, every
spilled slot is back before its W, and the pools never overflow.  Infeasible
budgets are refused (ENOMEM), never mis-planned."""
import ctypes as C

import pytest
from hypothesis import given, settings, strategies as st

import synthetic as sy
from paper_2504_19232_b200 import _lib as L
from paper_2504_19232_b200 import sched as cs
from paper_2504_19232_b200.pipeline import Arm


def plan(order, N, D, H, window=4, merge=False):
    n = len(order)
    arr = (L.Op * max(1, n))()
    for q, (k, mb) in enumerate(order):
        arr[q].kind, arr[q].mb = cs.KIND_ID[k], mb
    slots = (C.c_int32 * max(1, n))()
    cap = 4 * N + 8
    acts = (C.c_int32 * (6 * cap))()
    na = C.c_int32()
    rc = L.lib().adaptra_offload_plan(arr, n, N, D, H, window, L.MERGE_W if merge else 0, slots, acts, cap,
                                      C.byref(na))
    if rc == L.ENOMEM:
        return None
    L.check(rc)
    return list(slots[:n]), [tuple(acts[6 * k:6 * k + 6]) for k in range(na.value)]


def simulate(order, N, D, H, slots, acts, merge=False):
    dev = {}            # device slot -> mb holding it
    host = {}           # host slot -> mb
    where = {}          # mb -> ("dev", slot) | ("host", slot)
    b_done, w_pos = set(), {}
    after = {}
    for a in acts:
        after.setdefault(a[4], []).append(a)
    for q, (k, mb) in enumerate(order):
        if k == "W" or (merge and k == "B"):
            w_pos[mb] = q
    for q, (k, mb) in enumerate(order):
        s = slots[q]
        assert 0 <= s < D
        if k == "F":
            assert mb not in where
            assert s not in dev, f"F{mb} at {q}: slot {s} still holds {dev.get(s)}"
            dev[s] = mb
            where[mb] = ("dev", s)
        else:
            assert where.get(mb) == ("dev", s), (q, k, mb, where.get(mb), s)
            if k == "B":
                b_done.add(mb)
            if k == "W" or merge:
                del dev[s]
                del where[mb]
        for spill, m, dslot, hslot, aq, wq in after.get(q, []):
            assert wq > q
            if spill:
                assert m in b_done and where.get(m) == ("dev", dslot) and w_pos[m] > q
                assert hslot not in host and 0 <= hslot < H
                host[hslot] = m
                del dev[dslot]
                where[m] = ("host", hslot)
            else:
                assert where.get(m) == ("host", hslot) and dslot not in dev and 0 <= dslot < D
                assert wq == w_pos[m]
                del host[hslot]
                dev[dslot] = m
                where[m] = ("dev", dslot)
    assert not dev and not host and not where


def min_device_slots(order):
    """Only complete slots (B done) can leave the device, so it must hold every
    incomplete forward at each F, and those plus the slot a W brings back."""
    f = b = p = 0
    for k, _ in order:
        if k == "W":
            p = max(p, f - b + 1)
        f += k == "F"
        b += k == "B"
        p = max(p, f - b)
    return max(p, 1)


@st.composite
def cases(draw):
    S = draw(st.integers(2, 8))
    N = draw(st.integers(2, 32))
    seed = draw(st.integers(0, 10 ** 6))
    tF, tB, tW, _ = sy.stage_profile(seed, S, 1, 40)
    arm = draw(st.sampled_from(["zb", "1f1b", "adaptive"]))
    c = sy.stage_profile(seed + 1, S, 1, 2, draw(st.sampled_from([0, 30, 200])))[3]
    a = Arm(arm, S, N, tF, tB, tW)
    orders = a.plan(c)
    i = draw(st.integers(0, S - 1))
    extra = draw(st.integers(0, 3))
    return orders[i], N, a.merge_w, extra, draw(st.integers(1, 6))


@settings(max_examples=300, deadline=None)
@given(cases())
def test_offload_plan_is_valid(case):
    order, N, merge, extra, window = case
    D = min_device_slots(order) + extra
    got = plan(order, N, D, N, window, merge)
    assert got is not None, "that budget and a full host pool must be feasible"
    slots, acts = got
    simulate(order, N, D, N, slots, acts, merge)
    if D >= N:
        assert acts == []         # everything fits: no copies


def test_offload_plan_refuses_infeasible_budgets():
    t = [10] * 4
    order = Arm("zb", 4, 8, t, t, t).plan([0, 0, 0])[0]   # stage 0: 7 forwards before the first B
    assert plan(order, 8, 3, 8) is None                  # only complete slots can move
    assert plan(order, 8, 7, 0) is None                   # no host pool, peak F-W demand is 8
    # W1 brings slot 1 back while every device slot is taken: slot 2 (B done)
    # must go out first, so a swap needs two host slots
    assert plan(order, 8, 7, 1) is None
    ok = plan(order, 8, 7, 2)
    assert ok is not None
    simulate(order, 8, 7, 2, *ok)
