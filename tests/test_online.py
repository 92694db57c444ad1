"""Online straggler detection: the quantiser's pins, and the lag-1
planner's decisions on noisy measured latencies are the oracle's R18 policy +
Alg. 2 + R26 clamp + Schedule() (oracle.sched.adaptive_orders) applied to the
lagged, quantised sequence -- bit-identical orders and warm-up counts."""
import random

import pytest

from oracle import sched as sc
import synthetic as sy
import bench
from paper_2504_19232_b200.online import OnlinePlanner, quantize
from paper_2504_19232_b200.pipeline import Arm


def test_quantize_threshold_grid_hysteresis():
    t = 8000
    # below 0.1 t: noise -> 0
    assert quantize([799, 0], t) == [0, 0]
    # snaps to the 0.125 t grid (1000 ns), at least one step
    assert quantize([800, 2600], t) == [1000, 3000]
    # keeps the previous grid value while within half a step of it ...
    assert quantize([3400, 2550], t, prev=[3000, 3000]) == [3000, 3000]
    # ... and moves once it leaves that band
    assert quantize([3600, 2400], t, prev=[3000, 3000]) == [4000, 2000]
    # back to nominal releases the held value
    assert quantize([100, 0], t, prev=[3000, 3000]) == [0, 0]


@pytest.mark.parametrize("S,N,seed,hold", [(8, 32, 0, 3), (4, 16, 1, 2), (8, 32, 2, 1)])
def test_online_planner_matches_oracle_on_lagged_quantised_sequence(S, N, seed, hold):
    tF, tB, tW, _ = sy.stage_profile(seed, S, 4000, 9000)
    tF, tB, tW = [v * 1000 for v in tF], [v * 1000 for v in tB], [v * 1000 for v in tW]
    t_ref = sum(tF) // S
    host_c = 330_000
    x_cap = [N - i for i in range(S)]
    x_init = sc.clamp_plan(sc.get_init_warmup_fwds(S, x_cap[0], 1, N), x_cap)
    rng = random.Random(seed)
    injected, downs = [], []
    for ev in sy.PAPER_TRACE:
        c, down = bench.trace_c(ev, S, t_ref, host_c)
        for _ in range(hold):
            injected.append(c)
            downs.append(down)
        for _ in range(hold):
            injected.append([0] * (S - 1))
            downs.append([])
    planner = OnlinePlanner(Arm("adaptive", S, N, tF, tB, tW, x_init=x_init, x_cap=x_cap), t_ref)
    used_c, got = [], []
    for c, down in zip(injected, downs):
        used_c.append(list(planner.c_q))        # what iteration k is planned with (measured in k-1)
        orders = planner.orders()
        got.append((list(planner.x), orders))
        # the gate's measurement: injected latency + polling overhead and jitter;
        # a down link measures ~0 at the gate (timed after the D2H copy)
        meas = [0 if link in down else (int(v * (1 + rng.uniform(-0.03, 0.03))) + 15_000 if v else rng.randint(0, 200))
                for link, v in enumerate(c)]
        planner.observe(meas, down=down, host_c=host_c)
    # lag 1: iteration 0 is planned at nominal, iteration k with iteration k-1's quantised measurement
    assert used_c[0] == [0] * (S - 1)
    assert used_c[1:] == [h["quantized"] for h in planner.history[:-1]]
    ref = sc.adaptive_orders(S, N, tF, tB, tW, used_c, x_init, x_cap)
    for k, ((x_ref, order_ref), (x_got, order_got)) in enumerate(zip(ref, got)):
        assert x_got == x_ref, k
        assert order_got == order_ref, k
    # detection: every straggling link is seen (quantised > 0) one iteration late, nominal links stay 0
    for k in range(1, len(injected)):
        q = used_c[k]
        for link, v in enumerate(injected[k - 1]):
            if v > 0.1 * t_ref:
                assert q[link] > 0
            elif link not in downs[k - 1]:
                assert q[link] == 0


class _FakePipe:
    """Stands in for a Pipeline: only the attributes LinkMonitor reads."""

    def __init__(self, S, out_fwd, out_bwd):
        self.S, self.out_fwd, self.out_bwd = S, out_fwd, out_bwd


def test_link_monitor_pools_directions_and_ranks():
    """Per link: (sum of both directions' delays) / (their message count) over
    the interval since the previous sample, merged across ranks; max of the
    maxima; a link without gated messages measures 0 (R32, R16)."""
    from paper_2504_19232_b200 import online

    # two "ranks": rank A owns stage 0..1 outboxes, rank B stages 2..3 (S = 4)
    stats = {"A": {("fwd", 0): (0, 0, 0), ("fwd", 1): (0, 0, 0), ("bwd", 0): (0, 0, 0)},
             "B": {("bwd", 1): (0, 0, 0), ("bwd", 2): (0, 0, 0), ("fwd", 2): (0, 0, 0)}}
    mons = {}
    for r in ("A", "B"):
        m = online.LinkMonitor.__new__(online.LinkMonitor)
        m.pipe, m.S = _FakePipe(4, {}, {}), 4
        m._read = (lambda rr: (lambda: dict(stats[rr])))(r)
        m._last = m._read()
        mons[r] = m
    # interval: link 0 fwd 4 msgs x 1000 ns (rank A); link 0 bwd 4 msgs x 3000 ns (rank B's stage 1 outbox)
    #           link 1 fwd 2 msgs x 500, max 700 (rank A); link 2: nothing gated
    stats["A"][("fwd", 0)] = (4, 4000, 1000)
    stats["B"][("bwd", 0)] = (4, 12000, 3000)
    stats["A"][("fwd", 1)] = (2, 1000, 700)
    parts = {}
    for r in ("A", "B"):
        cur = mons[r]._read()
        parts[r] = {k: (v[0] - mons[r]._last.get(k, (0, 0, 0))[0], v[1] - mons[r]._last.get(k, (0, 0, 0))[1], v[2])
                    for k, v in cur.items()}
    gather = lambda _o: [parts["A"], parts["B"]]
    m = mons["A"]
    m.gather = gather
    m._read = lambda: dict(stats["A"])
    mean, mx = m.sample()
    assert mean == [2000, 500, 0]        # (4000 + 12000) / 8 ; 1000 / 2 ; none
    assert mx == [3000, 700, 0]
