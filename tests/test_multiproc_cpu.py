"""World-size-2 gloo test of the multi-process control plane on CPU: stage
placement, profile all-gather, and that every rank derives the bit-identical
schedule (R29) for every trace event, so no schedule broadcast is needed."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import synthetic as sy


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, S, N, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_19232_b200.pipeline import Arm
        import bench
        stage_rank = [i * world // S for i in range(S)]
        local = [i for i in range(S) if stage_rank[i] == rank]
        # each rank "measures" its own stages; all-gather gives everyone the full profile
        loc = {i: [1000 * (10 + i), 1000 * (11 + i), 1000 * 9] for i in local}
        out = [None] * world
        dist.all_gather_object(out, loc)
        prof = {}
        for d in out:
            prof.update(d)
        tF = [prof[i][0] for i in range(S)]
        tB = [prof[i][1] for i in range(S)]
        tW = [prof[i][2] for i in range(S)]
        arm = Arm("adaptive", S, N, tF, tB, tW)
        t_ref = sum(tF) // S
        plans = []
        for ev in sy.PAPER_TRACE:
            c, down = bench.trace_c(ev, S, t_ref, 500_000)
            plans.append((arm.plan(c), arm.x, down))
        allp = [None] * world
        dist.all_gather_object(allp, plans)
        q.put((rank, local, allp[0] == allp[1], arm.replans))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("S,N", [(4, 16), (8, 32)])
def test_two_ranks_agree_on_every_schedule(S, N):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, S, N, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == list(range(S // 2)) and res[1][1] == list(range(S // 2, S))
    assert all(r[2] for r in res)
    assert res[0][3] == res[1][3] and res[0][3] > 0
