"""Bit-exact parity of the C++ scheduling core (libadaptra.so, host code) with
the CPU oracle on the same integer inputs: plans, Eq. 1, every per-stage op
order with start/end times, makespan, step count, replay and validation.
Also checks that the library loads and exports every declared symbol."""
import ctypes

import pytest
from hypothesis import given, settings, strategies as st

from oracle import sched as sc
import synthetic as sy
from paper_2504_19232_b200 import _lib as L
from paper_2504_19232_b200 import sched as cs


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    header = open(L.HERE + "/../include/adaptra.h").read()
    import re
    declared = set(re.findall(r"\b(adaptra_[A-Za-z0-9_]+)\s*\(", header))
    declared = {d for d in declared if not d.endswith("_t")}
    assert declared == set(L.declared_symbols()), declared ^ set(L.declared_symbols())
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.adaptra_version().startswith(b"adaptra")


def _ox(X):
    return [[(o.kind, o.mb, o.start, o.end) for o in ops] for ops in X]


def test_pinned_cases_match():
    t = [10] * 4
    for c in ([0, 0, 0], [10, 0, 0], [20, 0, 0], [0, 0, 35]):
        for x in ([7, 5, 3, 1], [12, 8, 4, 1], [4, 3, 2, 1]):
            for mode in ("paper", "cap"):
                Xo, To, so = sc.schedule(4, 12, t, t, t, c, x, 1, mode=mode)
                Xc, Tc, s_c = cs.schedule(4, 12, t, t, t, c, x, 1, mode=mode)
                assert (To, so, _ox(Xo)) == (Tc, s_c, Xc)


@st.composite
def specs(draw):
    S = draw(st.integers(2, 8))
    N = draw(st.integers(1, 24))
    seed = draw(st.integers(0, 10 ** 9))
    c_hi = draw(st.sampled_from([0, 4, 20, 100, 400]))
    tF, tB, tW, c = sy.stage_profile(seed, S, 1, 40, c_hi)
    return S, N, tF, tB, tW, c, draw(st.integers(0, 2)), draw(st.integers(1, 7)), draw(st.booleans())


@settings(max_examples=400, deadline=None)
@given(specs())
def test_random_parity(spec):
    S, N, tF, tB, tW, c, plan, delta, cap = spec
    assert cs.plan_adapt(S, N, tF, tB, c) == sc.get_adapted_warmup_fwds(S, N, tF, tB, c)
    mem = (tF[0] * 7 + N) % 50 + 1
    assert cs.plan_init(S, N, mem, 1) == sc.get_init_warmup_fwds(S, mem, 1, N)
    if plan == 0:
        x = sc.get_adapted_warmup_fwds(S, N, tF, tB, c)
    elif plan == 1:
        x = sc.plan_1f1b(S, N)
    else:
        x = [max(1, v) for v in sc.get_init_warmup_fwds(S, mem, 1, N)]
        x = [min(v, x[0]) for v in x]
    assert cs.eq1_holds(tF, tB, c, x) == sc.eq1_holds(tF, tB, c, x)
    mode = "cap" if cap else "paper"
    for merge in (False, True):
        Xo, To, so = sc.schedule(S, N, tF, tB, tW, c, x, delta, mode=mode, merge_w=merge)
        Xc, Tc, s_c = cs.schedule(S, N, tF, tB, tW, c, x, delta, mode=mode, merge_w=merge)
        assert (To, so) == (Tc, s_c)
        assert _ox(Xo) == Xc
        assert cs.validate(S, N, tF, tB, tW, c, Xc, merge) == []
        # under other latencies the same timing is invalid in the same places on both sides
        c3 = [v + 3 for v in c]
        assert sorted(cs.validate(S, N, tF, tB, tW, c3, Xc, merge)) == sorted(
            sc.violations(S, N, tF, tB, tW, c3, Xo, merge))
        # replay under other latencies
        c2 = [v * 3 + 5 for v in c]
        Ro, RTo = sc.replay(S, N, tF, tB, tW, c2, sc.order_of(Xo), merge_w=merge)
        Rc, RTc = cs.replay(S, N, tF, tB, tW, c2, cs.order_of(Xc), merge_w=merge)
        assert RTo == RTc and _ox(Ro) == Rc


def test_errors():
    t = [10] * 4
    with pytest.raises(L.AdaptraError) as e:
        cs.schedule(4, 12, t, t, t, [0, 0, 0], [1, 3, 3, 1], 1)
    assert e.value.code == L.EPLAN
    with pytest.raises(L.AdaptraError) as e:
        cs.plan_init(1, 4, 4, 1)
    assert e.value.code == L.EINVAL
    with pytest.raises(L.AdaptraError) as e:
        cs.replay(2, 1, [1, 1], [1, 1], [1, 1], [0], [[("B", 1)], [("F", 1), ("B", 1)]])
    assert e.value.code == L.EDEADLOCK
    # a schedule with a dependency violation is flagged
    X, _, _ = cs.schedule(4, 12, t, t, t, [0, 0, 0], [7, 5, 3, 1], 1)
    bad = [list(s) for s in X]
    k, m, s0, e0 = bad[1][0]
    bad[1][0] = (k, m, s0 - 5, e0 - 5)
    assert ("dep", 1, "F", 1) in cs.validate(4, 12, t, t, t, [0, 0, 0], bad)


def _mutants():
    t = [10] * 4
    X, _, _ = sc.schedule(4, 12, t, t, t, [0, 0, 0], [7, 5, 3, 1], 1)
    base = [[(o.kind, o.mb, o.start, o.end) for o in ops] for ops in X]
    out = []
    m = [list(s) for s in base]; m[1][-1] = m[1][4][:2] + (m[1][-1][2], m[1][-1][3]); out.append(m)  # dup + missing
    m = [list(s) for s in base]; m[3].pop(); out.append(m)
    m = [list(s) for s in base]; k, j, a, b = m[2][-1]; m[2][-1] = (k, j, a, b + 1); out.append(m)
    m = [list(s) for s in base]; k, j, a, b = m[0][1]; m[0][1] = (k, j, a - 1, b - 1); out.append(m)
    m = [list(s) for s in base]; m[1][-1] = ("F", 13) + m[1][-1][2:]; out.append(m)
    m = [list(s) for s in base]; m[2] = m[2][::-1]; out.append(m)
    return out


@pytest.mark.parametrize("k", range(6))
def test_validate_violation_lists_match_oracle(k):
    """adaptra_validate returns the same violation list (as a multiset) as
    oracle.sched.violations on mutated copies of the ideal ZB schedule."""
    t = [10] * 4
    m = _mutants()[k]
    for c in ([0, 0, 0], [1, 0, 2]):
        got = cs.validate(4, 12, t, t, t, c, m)
        ref = sc.violations(4, 12, t, t, t, c, [[sc.Op(*o) for o in ops] for ops in m])
        assert got and sorted(got) == sorted(ref)
    # capacity: the total is reported even when the list is cut
    assert len(cs.validate(4, 12, t, t, t, [0, 0, 0], m, cap=1)) == 1


def test_validate_plan_matches_oracle():
    for N, x in ((12, [7, 5, 3, 1]), (12, [3, 4, 1]), (12, [5, 3, 3, 4]), (4, [5, 3, 1]), (12, [3, 2, 0]),
                 (2, [1, 3, 0])):
        assert sorted(cs.validate_plan(len(x), N, x)) == sorted(sc.plan_violations(N, x))


@st.composite
def arm_specs(draw):
    S = draw(st.integers(2, 8))
    N = draw(st.integers(1, 40))
    seed = draw(st.integers(0, 10 ** 9))
    tF, tB, tW, _ = sy.stage_profile(seed, S, 1, 60)
    cs_seq = []
    for k in range(draw(st.integers(1, 8))):
        c_hi = draw(st.sampled_from([0, 0, 10, 60, 300]))
        cs_seq.append(sy.stage_profile(seed + k + 1, S, 1, 2, c_hi)[3])
    cap = draw(st.sampled_from([None, 3, 8]))
    x_cap = None if cap is None else [max(1, cap - i // 2) for i in range(S)]
    return S, N, tF, tB, tW, cs_seq, x_cap, draw(st.sampled_from([10, 30]))


@settings(max_examples=150, deadline=None)
@given(arm_specs())
def test_planner_arms_match_oracle(spec):
    """adaptra_planner (R18 / R21 / R26 in C) == the oracle's baselines and
    adaptive_orders, iteration by iteration: plan and per-stage order."""
    S, N, tF, tB, tW, cs_seq, x_cap, ratio = spec
    zero = [0] * (S - 1)
    d = sc.default_delta(tF, tB, tW, ratio)
    assert cs.default_delta(tF, tB, tW, ratio) == d
    X1, _, _ = sc.schedule_1f1b(S, N, tF, tB, tW, d)
    Xz, _, _ = sc.schedule(S, N, tF, tB, tW, zero, sc.get_adapted_warmup_fwds(S, N, tF, tB, zero), d)
    for name, ref in (("1f1b", sc.order_of(X1)), ("zb", sc.order_of(Xz))):
        p = cs.Planner(name, S, N, tF, tB, tW, ratio=ratio)
        for c in cs_seq:                      # frozen: the latencies change nothing
            assert p.step(c)[0] == ref
    x_init = sc.get_init_warmup_fwds(S, 40, 1, N)
    if x_cap:
        x_init = sc.clamp_plan(x_init, x_cap)
    ref = sc.adaptive_orders(S, N, tF, tB, tW, cs_seq, x_init, x_cap, ratio)
    p = cs.Planner("adaptive", S, N, tF, tB, tW, x_cap=x_cap, mem=(40, 1), ratio=ratio)
    for (x_ref, order_ref), c in zip(ref, cs_seq):
        orders, x, _ = p.step(c)
        assert (x, orders) == (x_ref, order_ref)


def test_generation_latency_under_100ms():
    """P14: < 100 ms per generation at S=8, N=32, t_o/delta = 30."""
    import time
    S, N = 8, 32
    t = [2_500_000] * S        # 2.5 ms in ns
    c = [0, 0, 25_000_000, 0, 0, 0, 0]
    d = sc.default_delta(t, t, t)
    x = cs.plan_adapt(S, N, t, t, c)
    t0 = time.perf_counter()
    cs.schedule(S, N, t, t, t, c, x, d)
    assert time.perf_counter() - t0 < 0.1
