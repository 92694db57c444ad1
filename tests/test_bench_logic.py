"""Host logic of the bench's straggler trace (no GPU): the R27 link mapping for
pipelines shorter than the paper's 8 stages and the R22 latency scaling."""
import math

import bench
import synthetic as sy


def test_trace_links_r27():
    # 8 stages: the paper's links unchanged
    assert bench.trace_links([0, 5], 8) == [0, 5]
    # S stages: link a -> floor(a (S-1) / 7); duplicates merge
    assert bench.trace_links([2, 3, 6], 4) == [0, 1, 2]
    assert bench.trace_links([0, 1, 2], 4) == [0]
    assert bench.trace_links([6], 2) == [0]
    for S in (2, 3, 4, 5, 6, 7):
        for a in range(7):
            (m,) = bench.trace_links([a], S)
            assert 0 <= m <= S - 2


def test_trace_c_r22_scaling_and_failure():
    t_ref = 1_500_000          # measured stage t_F (ns)
    host_c = 330_000           # measured delegated-path latency (ns)
    ev = {"links": [2], "latency_ms": 30}
    c, down = bench.trace_c(ev, 8, t_ref, host_c)
    # latency_ms is in units of the paper's t = 10 ms: 30 ms -> 3 t_F
    assert c == [0, 0, 3 * t_ref, 0, 0, 0, 0] and down == []
    c, down = bench.trace_c({"links": [2], "latency_ms": math.inf}, 8, t_ref, host_c)
    assert down == [2] and c[2] == host_c and sum(c) == host_c
    # every event of the paper's trace maps to finite latencies on valid links
    for e in sy.PAPER_TRACE:
        for S in (4, 8):
            c, down = bench.trace_c(e, S, t_ref, host_c)
            assert len(c) == S - 1 and all(v >= 0 for v in c)
            assert all(0 <= l < S - 1 for l in down)
