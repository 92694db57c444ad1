"""Whole pipelined iteration (all stages co-located on cuda:0, one executor
thread per stage, mailboxes + flags, latency gate, delegated host path) vs
the oracle's unpipelined full-batch loss and gradients (P12), for every arm."""
import time

import numpy as np
import pytest
import torch

from oracle import numerics as nu
import synthetic as sy
from paper_2504_19232_b200 import _lib as L
from paper_2504_19232_b200.pipeline import Arm, ModelCfg, Pipeline

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def _setup(kind, dtype, S, N, Lt, d, dff, H, b, T, **kw):
    bf = dtype == L.BF16
    Ls = Lt // S
    params = (sy.mlp_params(0, S, Ls, d, dff, bf16=bf) if kind == "mlp"
              else sy.gpt_params(0, S, Ls, d, dff, perturb=True, bf16=bf))
    xs = sy.microbatches(1, N, b, T, d, bf16=bf)
    tg = sy.targets(2, N, b, T, d)
    m = ModelCfg(block=kind, n_layers=Lt, d=d, d_ff=dff, n_heads=H or 1, b=b, T=T, dtype=dtype)
    pipe = Pipeline(m, S, N, params=params, inputs=xs, targets=tg, **kw)
    Lref, gref, _ = nu.full_batch(kind, params, xs, tg, H)
    return pipe, Lref, gref


def _check(pipe, res, Lref, gref, tol):
    assert abs(res.loss - Lref) <= tol * abs(Lref), (res.loss, Lref)
    for i, st in pipe.stages.items():
        got = st.grads()
        for l in range(len(got)):
            for k in gref[i][l]:
                e = rel(got[l][k], gref[i][l][k])
                assert e < tol, (i, l, k, e)


CFGS = [
    # C0 (S=4, N=8, 2-layer MLP per stage hidden=64, fp32)
    ("mlp", L.F32, 4, 8, 4, 64, 64, None, 1, 32, 1e-4),
    ("gpt", L.BF16, 2, 4, 4, 256, 1024, 2, 1, 128, 2e-2),
]


@pytest.mark.parametrize("arm", ["1f1b", "zb", "adaptive", "zb-inorder", "1f1b-inorder"])
@pytest.mark.parametrize("kind,dtype,S,N,Lt,d,dff,H,b,T,tol", CFGS)
def test_pipeline_iteration_matches_full_batch(kind, dtype, S, N, Lt, d, dff, H, b, T, tol, arm):
    pipe, Lref, gref = _setup(kind, dtype, S, N, Lt, d, dff, H, b, T)
    try:
        t = [1000] * S
        a = Arm(arm, S, N, t, t, t)
        c = [0] * (S - 1)
        if arm == "adaptive":
            c[S // 2 - 1] = 2_000_000       # 2 ms injected on one link
            pipe.set_latency(S // 2 - 1, c[S // 2 - 1])
        orders = a.plan(c)
        for _ in range(2):                  # twice: epochs / mailbox reuse / zeroed grads
            res = pipe.run(orders, merge_w=a.merge_w, want_times=True, inorder=a.inorder)
        _check(pipe, res, Lref, gref, tol)
        for i, st in res.stats.items():
            assert st["op_cnt"][0] == N
            times = st["op_times"]
            assert all(times[q][0] >= times[q - 1][1] - 1000 for q in range(1, len(times)))
    finally:
        pipe.close()


@pytest.mark.parametrize("mode", [L.LINK_DIRECT, L.LINK_P2P])
def test_latency_injection_and_link_down(mode):
    S, N = 4, 8
    pipe, Lref, gref = _setup("mlp", L.F32, S, N, 4, 64, 64, None, 1, 32, link_mode=mode)
    try:
        t = [1000] * S
        a = Arm("zb", S, N, t, t, t)
        orders = a.plan([0] * (S - 1))
        base = pipe.run(orders, want_times=True)
        # 5 ms on link 1: stage 2's first F cannot start before stage 1's first F ends + 5 ms
        pipe.set_latency(1, 5_000_000)
        res = pipe.run(orders, want_times=True)
        f1_end = res.stats[1]["op_times"][0][1]
        f2_start = res.stats[2]["op_times"][0][0]
        assert f2_start - f1_end >= 4_900_000, (f1_end, f2_start)
        _check(pipe, res, Lref, gref, 1e-4)
        n, s, m = pipe.link_stats()[("fwd", 1)]
        assert n >= N and s / n >= 4_900_000
        # link 1 fails: traffic moves to the delegated host path, results unchanged
        pipe.set_latency(1, L.LINK_DOWN)
        res = pipe.run(orders)
        _check(pipe, res, Lref, gref, 1e-4)
        pipe.set_latency(1, 0)
        res = pipe.run(orders)
        _check(pipe, res, Lref, gref, 1e-4)
        # delegation policy: a straggling (up) link moved to the host path keeps
        # its latency and the results
        pipe.set_latency(1, 3_000_000)
        pipe.set_path(1, True)
        res = pipe.run(orders, want_times=True)
        _check(pipe, res, Lref, gref, 1e-4)
        assert res.stats[2]["op_times"][0][0] - res.stats[1]["op_times"][0][1] >= 2_900_000
        pipe.set_path(1, False)
        pipe.set_latency(1, 0)
        res = pipe.run(orders)
        _check(pipe, res, Lref, gref, 1e-4)
    finally:
        pipe.close()


def test_pipeline_full_size_c1_layers():
    """The whole pipelined iteration at C1 sizes (d=2048, 16 heads, d_ff=8192,
    T=2048, bf16): 2 stages x 2 layers, N=2, adaptive arm with 2 ms injected on
    the link -- producer epilogues storing into the peer mailbox, fused
    attention, grouped dW launches -- vs the fp64 full batch (P12, 2e-2)."""
    S, N, Lt, d, dff, H, b, T = 2, 2, 4, 2048, 8192, 16, 1, 2048
    pipe, Lref, gref = _setup("gpt", L.BF16, S, N, Lt, d, dff, H, b, T)
    try:
        t = [1_000_000] * S
        a = Arm("adaptive", S, N, t, t, t)
        c = [2_000_000]
        pipe.set_latency(0, c[0])
        orders = a.plan(c)
        res = pipe.run(orders, merge_w=a.merge_w, want_times=True)
        _check(pipe, res, Lref, gref, 2e-2)
    finally:
        pipe.set_latency(0, 0)
        pipe.close()


def test_host_io_end_to_end_matches_device_path():
    """adaptra_exec_set_host_io: inputs uploaded from pinned host buffers by the
    executor every iteration and the loss copied back to the host give the
    same loss (bit for bit: fixed-order reduction) and gradients as the
    device-resident run, and the profiler (adaptra_exec_profile, a1) reports
    every kind's median op time."""
    S, N = 2, 4
    pipe, Lref, gref = _setup("gpt", L.BF16, S, N, 4, 256, 1024, 2, 1, 128)
    try:
        t = [1000] * S
        a = Arm("zb", S, N, t, t, t)
        orders = a.plan([0])
        dev = pipe.run(orders).loss
        h2d, d2h = pipe.set_host_io(True)   # pinned host copies of the inputs
        for t_ in pipe.inputs:              # the device copies are rewritten by the uploads
            t_.zero_()
        torch.cuda.synchronize()
        assert h2d == N * 128 * 256 * 2 and d2h == 4
        for _ in range(3):
            res = pipe.run(orders)
        assert res.loss == dev
        _check(pipe, res, Lref, gref, 2e-2)
        tF, tB, tW = pipe.profile(k=3)
        assert all(v >= 1000 and v % 1000 == 0 for v in tF + tB + tW)
        pipe.set_host_io(False)
    finally:
        pipe.close()


@pytest.mark.parametrize("arm", ["zb", "adaptive"])
@pytest.mark.parametrize("kind,dtype,S,N,Lt,d,dff,H,b,T,tol", CFGS)
def test_stash_offload_matches_device_run(kind, dtype, S, N, Lt, d, dff, H, b, T, tol, arm):
    """N4: with as few device F->W slots per stage as the order
    allows (its peak in-flight forwards) and the rest in a pinned host pool (Belady spills after B, prefetch before W), the iteration
    gives the same loss and gradients as with every slot on the device (bit
    for bit) and as the oracle's full batch; the plan really spilled."""
    ref_pipe, Lref, gref = _setup(kind, dtype, S, N, Lt, d, dff, H, b, T)
    t = [1000] * S
    try:
        a = Arm(arm, S, N, t, t, t)
        c = [0] * (S - 1)
        if arm == "adaptive":
            c[0] = 3_000_000
            ref_pipe.set_latency(0, c[0])
        orders = a.plan(c)
        ref = ref_pipe.run(orders)
        ref_grads = {i: st.grads() for i, st in ref_pipe.stages.items()}
    finally:
        ref_pipe.close()
    # device slots per stage = the order's peak in-flight forwards (F - B):
    # only slots whose B is done can move to the host; the F->W demand is N
    peak = []                    # incomplete forwards (+ the slot a W brings back)
    for ops in orders:
        f = bb = p = 0
        for k, _ in ops:
            if k == "W":
                p = max(p, f - bb + 1)
            f += k == "F"
            bb += k == "B"
            p = max(p, f - bb)
        peak.append(max(p, 1))
    assert min(peak) < N
    pipe, _, _ = _setup(kind, dtype, S, N, Lt, d, dff, H, b, T, n_slots=peak)
    try:
        pipe.enable_offload(N, window=2)
        if arm == "adaptive":
            pipe.set_latency(0, c[0])
        for _ in range(2):
            res = pipe.run(orders)
        assert res.loss == ref.loss
        for i, st in pipe.stages.items():
            got = st.grads()
            for l in range(len(got)):
                for k in got[l]:
                    assert np.array_equal(got[l][k], ref_grads[i][l][k]), (i, l, k)
        _check(pipe, res, Lref, gref, tol)
        st = pipe.offload_stats()
        assert sum(v[0] for v in st.values()) > 0 and all(v[0] == v[1] for v in st.values())
    finally:
        pipe.close()


def test_bubble_metrics_match_oracle_definition():
    """a11 (R15): the bubble rates computed from an executed
    iteration's per-op CUDA-event times equal oracle.sched.metrics on the same
    times (utilisation and interior forms), under an injected straggler."""
    from oracle import sched as sc
    from paper_2504_19232_b200.pipeline import iteration_metrics
    S, N = 4, 8
    pipe, _, _ = _setup("gpt", L.BF16, S, N, 4, 256, 1024, 2, 1, 128)
    try:
        t = [1000] * S
        a = Arm("adaptive", S, N, t, t, t)
        c = [0, 3_000_000, 0]
        pipe.set_latency(1, c[1])
        orders = a.plan(c)
        res = pipe.run(orders, want_times=True)
        got = iteration_metrics(res.stats, orders)
        t0 = min(st["op_times"][0][0] for st in res.stats.values())
        X = [[sc.Op(k, mb, s - t0, e - t0) for (k, mb), (s, e) in zip(orders[i], res.stats[i]["op_times"])]
             for i in range(S)]
        ref = sc.metrics(S, X)
        assert ref["T"] == got["T_ns"] and ref["busy"] == got["busy_ns"]
        assert abs(ref["util_bubble"] - got["util_bubble"]) < 1e-12
        assert abs(ref["interior_bubble"] - got["interior_bubble"]) < 1e-12
        assert got["util_bubble"] > 0.0          # the 3 ms straggler leaves idle time
    finally:
        pipe.set_latency(1, 0)
        pipe.close()
