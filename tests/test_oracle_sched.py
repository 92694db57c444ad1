"""Pins for the schedule oracle (oracle/sched.py) against what the paper and
the mathematics fix (pins P1-P15).  CPU only."""
import json
import os

import pytest
from hypothesis import given, settings, strategies as st

from oracle import sched as sc
import synthetic as sy

GOLD = os.path.join(os.path.dirname(__file__), "golden")
T10 = [10] * 4


def _fixture_orders():
    rows = {}
    for line in open(os.path.join(GOLD, "ideal_zb_S4_N12.txt")):
        if line.startswith("#") or not line.strip():
            continue
        k, v = line.split(":")
        rows[int(k[1:])] = [(tok[0], int(tok[1:])) for tok in v.split()]
    return [rows[i] for i in range(4)]


def test_p1_ideal_zb_390ms_and_order():
    """P1: Fig. ideal_zb: T = 390 ms, zero interior bubbles."""
    gold = json.load(open(os.path.join(GOLD, "paper_values.json")))["ideal_zb"]
    x = sc.get_adapted_warmup_fwds(4, 12, T10, T10, [0, 0, 0])
    assert x == [7, 5, 3, 1]
    assert sc.get_init_warmup_fwds(4, 7, 1) == x
    for mode in (sc.MODE_PAPER, sc.MODE_CAP):
        X, T, steps = sc.schedule(4, 12, T10, T10, T10, [0, 0, 0], x, 1, mode=mode)
        assert T == gold["T_ms"]
        assert sc.order_of(X) == _fixture_orders()
        m = sc.metrics(4, X, T)
        assert m["interior_bubble"] == 0.0
        for i in range(4):
            assert X[i][0].start == 10 * i and X[i][-1].end == 360 + 10 * i
        assert steps == 381
        assert sc.validate(4, 12, T10, T10, T10, [0, 0, 0], X) == []


@pytest.mark.parametrize("key", ["delay_zb_10", "delay_zb_20"])
def test_p2_delayed_zb(key):
    """P2: Fig. delay_zb: the fixed ideal order under
    c_0 = 10 ms -> 400 ms; c_0 = 20 ms -> 440 ms with S_0's B_1 at 110 ms."""
    g = json.load(open(os.path.join(GOLD, "paper_values.json")))[key]
    X, T = sc.replay(4, 12, T10, T10, T10, g["c_ms"], _fixture_orders())
    assert T == g["T_ms"]
    assert sc.validate(4, 12, T10, T10, T10, g["c_ms"], X) == []
    if "stage0_B1_start_ms" in g:
        b1 = [op for op in X[0] if op.kind == "B" and op.mb == 1][0]
        assert b1.start == g["stage0_B1_start_ms"]


def test_p6_alg1_alg2_hand_traces():
    """P6/P8: hand executions of Alg. 1 and Alg. 2."""
    assert sc.get_init_warmup_fwds(4, 7, 1) == [7, 5, 3, 1]
    assert sc.get_init_warmup_fwds(4, 8, 1) == [8, 5, 3, 1]    # Delta_avg=2, r=1
    assert sc.get_init_warmup_fwds(2, 1, 1) == [1, 1]
    assert sc.get_init_warmup_fwds(4, 100, 3, N=12) == [12, 8, 4, 1]  # R12 clamp to N (11//3=3, r=2)
    assert sc.get_adapted_warmup_fwds(4, 12, T10, T10, [20, 0, 0]) == [8, 5, 3, 1]
    assert sc.get_adapted_warmup_fwds(4, 12, T10, T10, [100, 0, 0]) == [9, 5, 3, 1]  # clip N-2S=4
    assert sc.get_adapted_warmup_fwds(4, 12, T10, T10, [0, 0, 20]) == [8, 6, 4, 1]
    # R11: N < 2S floors Delta at 0
    assert sc.get_adapted_warmup_fwds(4, 6, T10, T10, [0, 0, 0]) == [1, 1, 1, 1]
    with pytest.raises(sc.PlanError):
        sc.get_init_warmup_fwds(1, 4, 1)
    with pytest.raises(sc.PlanError):
        sc.get_init_warmup_fwds(3, 0, 1)


def test_p7_eq1_boundaries():
    """Eq. 1 at its boundary (uniform t=10, Delta=2: c <= 10)."""
    x = [7, 5, 3, 1]
    assert sc.eq1_holds(T10, T10, [10, 0, 0], x) == [True, True, True]
    assert sc.eq1_holds(T10, T10, [11, 0, 0], x) == [False, True, True]
    # heterogeneous: tF_i=tB_i=10, tF_{i+1}=tB_{i+1}=20, Delta=1, c=10 -> 40 <= 40
    assert sc.eq1_holds([10, 20], [10, 20], [10], [2, 1]) == [True]
    assert sc.eq1_holds([10, 20], [10, 20], [11], [2, 1]) == [False]


def test_p4_1f1b_closed_form():
    """P4: 1F1B at c=0: T = (N+S-1)(tF+tB+tW), bubble = (S-1)/(N+S-1) (north_star)."""
    for S in range(2, 7):
        for N in range(1, 14):
            t = [10] * S
            X, T, _ = sc.schedule_1f1b(S, N, t, t, t, 1)
            assert T == (N + S - 1) * 30
            m = sc.metrics(S, X, T)
            assert abs(m["util_bubble"] - (S - 1) / (N + S - 1)) < 1e-12
            assert sc.validate(S, N, t, t, t, [0] * (S - 1), X, merge_w=True) == []
            # canonical 1F1B: warm-up S-i forwards then alternate
            assert m["warmup"] == [min(S - i, N) for i in range(S)]


def test_p5_zb_closed_form():
    """P5: ZB at c=0 with the Alg. 2 plan, N >= 2S: T = (S-1)tF + N(tF+tB+tW)."""
    for S in range(2, 7):
        for N in range(2 * S, 2 * S + 6):
            t = [10] * S
            X, T, _ = sc.schedule_zb(S, N, t, t, t, 1)
            assert T == (S - 1) * 10 + N * 30
            assert sc.metrics(S, X, T)["interior_bubble"] == 0.0


def test_p9_theorem1_regimes():
    """Theorem 1 in fixed-order replay, Delta in {1, 2}, t = 10:
    c <= (Delta-1)t -> accumulated delay exactly c, independent of N;
    c > (Delta-1)t -> grows linearly with N at 2(c-(Delta-1)t)/(Delta+1) per microbatch."""
    def acc(x, mode, c, N):
        X, T0, _ = sc.schedule(4, N, T10, T10, T10, [0] * 3, x, 1, mode=mode)
        _, T = sc.replay(4, N, T10, T10, T10, c, sc.order_of(X))
        return T - T0
    for link in (0, 2):
        c = [0, 0, 0]
        c[link] = 10
        assert acc([7, 5, 3, 1], sc.MODE_PAPER, c, 30) == 10 == acc([7, 5, 3, 1], sc.MODE_PAPER, c, 60)
        c[link] = 20
        slope = (acc([7, 5, 3, 1], sc.MODE_PAPER, c, 60) - acc([7, 5, 3, 1], sc.MODE_PAPER, c, 30)) / 30
        assert abs(slope - 2 * (20 - 10) / 3) < 1e-9
    for cv in (5, 20):
        c = [cv, 0, 0]
        slope = (acc([4, 3, 2, 1], sc.MODE_CAP, c, 60) - acc([4, 3, 2, 1], sc.MODE_CAP, c, 30)) / 30
        assert abs(slope - 2 * cv / 2) < 1e-9


def test_p10_adaptive_reaches_lower_bound_under_trace_events():
    """P10: for each multi-link event of the paper trace (t-scaled, R22), the
    Alg. 2 plan + Schedule reaches LB_c = sum(tF_i + c_i) + N(3t) exactly,
    while the frozen ZB and 1F1B orders do not."""
    S, N = 8, 32
    t = [10] * S
    d = sc.default_delta(t, t, t)
    X1, _, _ = sc.schedule_1f1b(S, N, t, t, t, d)
    Xz, _, _ = sc.schedule_zb(S, N, t, t, t, d)
    for ev in sy.PAPER_TRACE[:9]:
        c = [0] * (S - 1)
        for l in ev["links"]:
            c[l] = int(ev["latency_ms"])        # t = 10 ms units (R22)
        x = sc.get_adapted_warmup_fwds(S, N, t, t, c)
        X, T, _ = sc.schedule(S, N, t, t, t, c, x, 1)
        assert sc.validate(S, N, t, t, t, c, X) == []
        assert T == sc.lower_bound_c(S, N, t, t, t, c)
        _, Tz = sc.replay(S, N, t, t, t, c, sc.order_of(Xz))
        _, T1 = sc.replay(S, N, t, t, t, c, sc.order_of(X1), merge_w=True)
        assert T < Tz and T < T1


def test_p11_near_optimal_tiny():
    """P11 (< 1 % from the optimum): brute-force optimum on tiny
    instances; the heuristic with delta = t_o/30 stays close."""
    within1 = 0
    cases = 0
    for seed in range(8):
        S, N = 2, 3 if seed % 2 else 2
        tF, tB, tW, c = sy.stage_profile(seed, S, 5, 20, 15)
        delta = sc.default_delta(tF, tB, tW)
        x = sc.get_adapted_warmup_fwds(S, N, tF, tB, c)
        _, T, _ = sc.schedule(S, N, tF, tB, tW, c, x, delta)
        opt = sc.brute_force_optimum(S, N, tF, tB, tW, c)
        assert T >= opt
        cases += 1
        within1 += (T - opt) <= 0.01 * opt
        assert T <= 1.10 * opt
    assert within1 >= cases // 2


def test_spec_erratum_e1_two_stage_optimum():
    """S=2, N=2, t=10 -> 70 ms = the (S-1)t + 3Nt bound (not 80)."""
    t = [10, 10]
    X, T, _ = sc.schedule(2, 2, t, t, t, [0], sc.get_adapted_warmup_fwds(2, 2, t, t, [0]), 1)
    assert T == 70 == sc.brute_force_optimum(2, 2, t, t, t, [0])


def test_adaptive_policy_r18():
    x_init = [12, 8, 4, 1]
    x, r = sc.adaptive_plan(4, 12, T10, T10, [0, 0, 0], x_init, x_init)
    assert (x, r) == (x_init, False)
    x, r = sc.adaptive_plan(4, 12, T10, T10, [0, 0, 100], [7, 5, 3, 1], x_init)
    assert r and x == [9, 7, 5, 1]
    x2, r2 = sc.adaptive_plan(4, 12, T10, T10, [0, 0, 100], x, x_init)
    assert x2 == x  # Eq. 1 can fail only on the clipped link -> same plan, no change


# --------------------------------------------------------------------------
# Properties over random instances
# --------------------------------------------------------------------------

@st.composite
def instances(draw):
    S = draw(st.integers(2, 6))
    N = draw(st.integers(1, 14))
    seed = draw(st.integers(0, 10 ** 6))
    c_hi = draw(st.sampled_from([0, 5, 30, 80]))
    tF, tB, tW, c = sy.stage_profile(seed, S, 3, 20, c_hi)
    mode = draw(st.sampled_from([sc.MODE_PAPER, sc.MODE_CAP]))
    plan = draw(st.sampled_from(["adapt", "init", "1f1b"]))
    if plan == "adapt":
        x = sc.get_adapted_warmup_fwds(S, N, tF, tB, c)
    elif plan == "init":
        x = sc.get_init_warmup_fwds(S, draw(st.integers(1, 40)), 1, N)
        x = [max(1, v) for v in x]
        x = [min(v, x[0]) for v in x]
    else:
        x = sc.plan_1f1b(S, N)
    delta = draw(st.integers(1, 6))
    return S, N, tF, tB, tW, c, x, mode, delta


@settings(max_examples=150, deadline=None)
@given(instances())
def test_schedule_properties(inst):
    S, N, tF, tB, tW, c, x, mode, delta = inst
    assert sc.validate_plan(N, x) == []
    X, T, steps = sc.schedule(S, N, tF, tB, tW, c, x, delta, mode=mode)
    # dependency validity of every emitted schedule (north_star)
    assert sc.validate(S, N, tF, tB, tW, c, X) == []
    m = sc.metrics(S, X, T)
    # Lemma: measured warm-up counts non-increasing
    assert all(m["warmup"][i] >= m["warmup"][i + 1] for i in range(S - 1))
    assert 0.0 <= m["util_bubble"] <= 1.0 and 0.0 <= m["interior_bubble"] <= 1.0
    assert T >= sc.lower_bound_c(S, N, tF, tB, tW, c)
    # E7: steps <= ceil(T/delta) + 1 always
    assert steps <= -(-T // delta) + 1
    # replay of the emitted order under the same c is never later
    Xr, Tr = sc.replay(S, N, tF, tB, tW, c, sc.order_of(X))
    assert Tr <= T
    if delta == 1:
        assert Tr == T
    # determinism
    X2, T2, s2 = sc.schedule(S, N, tF, tB, tW, c, x, delta, mode=mode)
    assert (T2, s2, sc.order_of(X2)) == (T, steps, sc.order_of(X))


@settings(max_examples=100, deadline=None)
@given(st.integers(2, 8), st.integers(1, 40), st.integers(1, 50))
def test_plan_properties(S, N, xmax):
    x = sc.get_init_warmup_fwds(S, xmax, 1, N)
    d = sc.slackness(x)
    assert x[0] == min(xmax, N)
    if min(xmax, N) >= S:
        assert x[-1] == 1
        assert max(d) - min(d) <= 1
    tF, tB, tW, c = sy.stage_profile(S * 100 + N, S, 3, 20, 60)
    xa = sc.get_adapted_warmup_fwds(S, N, tF, tB, c)
    assert xa[-1] == 1 and all(xa[i] >= xa[i + 1] for i in range(S - 1)) and xa[0] <= N
    ok = sc.eq1_holds(tF, tB, c, xa)
    for i in range(S - 1):
        dl = xa[i] - xa[i + 1]
        # Either Eq. 1 holds or the clip (N-2S, or the R11 cap at N) is active
        assert ok[i] or dl == max(0, N - 2 * S) or xa[i] == N


def test_p13_bubble_formula():
    """R15: utilisation bubble 1 - sum(busy)/(S T).  The ideal ZB schedule
     has no interior gaps ("zero bubbles") and utilisation
    bubble 1/13; the paper's three (T, bubble) pairs of the 7B microbenchmark
    (ZB 703 ms / 57.4 %, Adaptra-CPU 579 / 48.8 %, Adaptra 398 / 25.3 %,
    S = 4) imply the same total busy time (about 1.19 s) only under this form."""
    X, T, _ = sc.schedule(4, 12, T10, T10, T10, [0, 0, 0], [7, 5, 3, 1], 1)
    m = sc.metrics(4, X, T)
    assert T == 390 and m["interior_bubble"] == 0.0
    assert abs(m["util_bubble"] - 1 / 13) < 1e-12
    busy = [4 * t * (1 - b) for t, b in ((703, 0.574), (579, 0.488), (398, 0.253))]
    assert max(busy) / min(busy) < 1.015 and all(1180 < v < 1200 for v in busy)


def test_peak_activations_equal_the_plan():
    """Peak in-flight forwards per stage (max over time of #F - #B) equals the
    warm-up plan on the ideal ZB timeline ([7, 5, 3, 1]) and on an adapted
    plan ([9, 5, 3, 1]) at c = 0 (SPEC peak_activations examples, derived)."""
    for x in ([7, 5, 3, 1], [9, 5, 3, 1]):
        X, T, _ = sc.schedule(4, 12, T10, T10, T10, [0, 0, 0], x, 1)
        assert sc.metrics(4, X, T)["peak_inflight"] == x
