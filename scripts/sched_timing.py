"""Schedule() generation time (P14; "< 100 ms"): the oracle
(Python) and the C++ core (adaptra_schedule through the C-ABI), 1 core each,
at the shapes of C1 (S=4, N=16), C2/C3 (S=8, N=32) and N=64, t_o/delta = 30,
uniform stage times and under one of the paper's trace events.  Host only.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import sched as osc  # noqa: E402
from paper_2504_19232_b200 import sched as cs  # noqa: E402
import synthetic as sy  # noqa: E402
import bench  # noqa: E402


def best(fn, reps):
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        t.append(time.perf_counter() - t0)
    return min(t) * 1e3


rows = []
for S, N in ((4, 16), (8, 32), (8, 64)):
    t = [1_500_000] * S
    delta = osc.default_delta(t, t, t, 30)
    for label, ev in (("nominal", None), ("trace event 3", sy.PAPER_TRACE[3])):
        c = [0] * (S - 1) if ev is None else bench.trace_c(ev, S, t[0], 330_000)[0]
        x = osc.get_adapted_warmup_fwds(S, N, t, t, c)
        o_ms = best(lambda: osc.schedule(S, N, t, t, t, c, x, delta), 3)
        c_ms = best(lambda: cs.schedule(S, N, t, t, t, c, x, delta), 20)
        X, T, steps = cs.schedule(S, N, t, t, t, c, x, delta)
        rows.append({"S": S, "N": N, "case": label, "delta_ns": delta, "steps": steps,
                     "oracle_python_ms": round(o_ms, 2), "cxx_ms": round(c_ms, 3),
                     "paper_budget_ms": 100, "speedup": round(o_ms / c_ms, 1)})
for r in rows:
    print(json.dumps(r))
