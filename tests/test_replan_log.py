""""schedules and per-stage op orders bit-exact vs the oracle
... including every re-plan logged during C2/C3".  The bench's adaptive arm
logs, per step on the B200, the integer inputs of its planning decision (the
profile t^F/t^B/t^W it used, c, the previous plan) and its outputs (x, delta,
the simulated makespan, every stage's op order); every logged step is
replayed here through the oracle (R18 policy, Alg. 1/2, R26 clamp, Schedule())."""
import glob
import json
import os

import pytest

from oracle import sched as sc

LOGS = sorted(glob.glob(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "profiles", "r*_replan_log_*.jsonl")))


def _orders(rows):
    return [[(tok[0], int(tok[1:])) for tok in row.split()] for row in rows]


def test_logs_exist():
    assert LOGS, "no committed re-plan log under profiles/"


@pytest.mark.parametrize("path", LOGS, ids=[os.path.basename(p) for p in LOGS])
def test_logged_replans_match_oracle(path):
    lines = [json.loads(l) for l in open(path) if l.strip()]
    head, steps = lines[0], lines[1:]
    S, N, x_cap, ratio = head["S"], head["N"], head["x_cap"], head["ratio"]
    x_init = sc.clamp_plan(sc.get_init_warmup_fwds(S, head["mem"][0], head["mem"][1], N), x_cap)
    assert head["x_init"] == x_init
    assert steps
    n_replans = 0
    for e in steps:
        tF, tB, tW, c = e["tF"], e["tB"], e["tW"], e["c"]
        x, order = sc.adaptive_step(S, N, tF, tB, tW, c, e["x_prev"], x_init, x_cap, ratio)
        assert x == e["x"], e["step"]
        assert order == _orders(e["orders"]), e["step"]
        delta = sc.default_delta(tF, tB, tW, ratio)
        assert delta == e["delta"]
        X, T, _ = sc.schedule(S, N, tF, tB, tW, c, x, delta)
        assert T == e["makespan"]
        assert sc.validate(S, N, tF, tB, tW, c, X) == []
        n_replans += e["replanned"]
    assert n_replans >= 1
