"""Every re-plan the bench's adaptive arm makes under the paper's straggler
trace (t-scaled as in bench.py, R22/R27) is bit-identical to the
oracle's R18 policy + Alg. 2 + R26 clamp + Schedule() on the same inputs."""
import pytest

from oracle import sched as sc
import synthetic as sy
import bench
from paper_2504_19232_b200.pipeline import Arm


@pytest.mark.parametrize("S,N,seed", [(8, 32, 0), (4, 16, 1), (8, 16, 2)])
def test_adaptive_arm_replans_match_oracle(S, N, seed):
    # stage op times shaped like the bench's measured ones (ns, 1 us quantised)
    tF, tB, tW, _ = sy.stage_profile(seed, S, 4000, 9000)
    tF, tB, tW = [v * 1000 for v in tF], [v * 1000 for v in tB], [v * 1000 for v in tW]
    t_ref = sum(tF) // S
    host_c = 330_000
    x_cap = [N - i for i in range(S)]
    x_init = sc.clamp_plan(sc.get_init_warmup_fwds(S, x_cap[0], 1, N), x_cap)
    cs_seq = []
    for k in range(25):
        ev = sy.PAPER_TRACE[k % len(sy.PAPER_TRACE)]
        c, _down = bench.trace_c(ev, S, t_ref, host_c)
        cs_seq.append(c)
        if k % 4 == 3:
            cs_seq.append([0] * (S - 1))   # back to nominal: revert to the init plan
    ref = sc.adaptive_orders(S, N, tF, tB, tW, cs_seq, x_init, x_cap)
    arm = Arm("adaptive", S, N, tF, tB, tW, x_init=x_init, x_cap=x_cap)
    for (x_ref, order_ref), c in zip(ref, cs_seq):
        orders = arm.plan(c)
        assert arm.x == x_ref
        assert orders == order_ref
