"""a1: the profiler's reduction, adaptra_median_ticks,
is the lower median floored to the tick quantum (at least one quantum) --
checked against statistics.median_low on random samples.  Host function, no GPU."""
import ctypes as C
import random
import statistics

from paper_2504_19232_b200 import _lib as L


def test_median_ticks_is_floored_lower_median():
    lib = L.lib()
    rng = random.Random(0)
    for n in range(1, 40):
        v = [rng.randrange(1, 5_000_000) for _ in range(n)]
        for q in (1, 1000, 7):
            got = lib.adaptra_median_ticks((C.c_int64 * n)(*v), n, q)
            assert got == max(q, statistics.median_low(v) // q * q)
    assert lib.adaptra_median_ticks((C.c_int64 * 1)(5), 1, 1000) == 1000   # at least one quantum
    assert lib.adaptra_median_ticks(None, 0, 1000) == -1
