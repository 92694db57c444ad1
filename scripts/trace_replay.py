"""Config C3: the paper's straggler trace (nine
multi-link latency events + a link failure from iteration 1030) replayed
iteration by iteration on 8 stages, compressed `--compress`x in time (1200 ->
120 iterations at 10x, labelled as such), for the arms
  adaptive  planner told the injected latencies (R18, lag 0)
  online    planner fed the transport's measured latencies (lag 1)
  zb        fixed ZB order (Alg. 2 plan at c = 0)
  1f1b      fixed 1F1B order
  zb-inorder / 1f1b-inorder  the same orders with blocking receives and a
            bounded send queue in the compute sequence
  zb-nccl / 1f1b-nccl  the same orders with real NCCL send/recv in the
            compute sequence (one stage per GPU; N1)
  adaptive-deleg  adaptive, straggling links moved to the delegated host path
on the same kernels and transport.  Latencies are scaled per R22 (latency_ms
in units of the paper's t = 10 ms, times the measured stage t_F); the failed
link carries its traffic on the delegated host path in every arm (the fixed
baselines of the paper would instead restart; that penalty is not charged).
One JSON line per arm (whole-trace tokens/s, mean bubble, replans) and one
per event (mean iteration time per arm) on rank 0.

  python -m torch.distributed.run --nproc-per-node 4 ... scripts/trace_replay.py [--S 8 --N 32]
"""
import argparse
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ["NCCL_DEBUG"] = "WARN"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--S", type=int, default=8)
    ap.add_argument("--N", type=int, default=32)
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--width", type=int, default=2048)
    ap.add_argument("--compress", type=int, default=10)
    ap.add_argument("--arms", default="adaptive,online,zb,1f1b")
    ap.add_argument("--replan-log", default="", help="JSONL of the first adaptive arm's per-iteration plans")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import bench
    import synthetic as sy
    from paper_2504_19232_b200 import _lib as L
    from paper_2504_19232_b200.online import LinkMonitor, OnlinePlanner
    from paper_2504_19232_b200.pipeline import Arm, ModelCfg, Pipeline

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        group = dist.new_group(backend="gloo")

    def gather(o):
        if world == 1:
            return [o]
        out = [None] * world
        dist.all_gather_object(out, o, group=group)
        return out

    S, N = args.S, args.N
    m = ModelCfg(block="gpt", n_layers=args.layers, d=args.width, d_ff=4 * args.width, n_heads=args.width // 128,
                 b=1, T=2048, dtype=L.BF16)
    pipe = Pipeline(m, S, N, rank=rank, world=world, device=local, group=group, host_links=True)
    prof = Arm("zb", S, N, [1000] * S, [1000] * S, [1000] * S)
    for _ in range(3):
        pipe.run(prof.orders)
    tF, tB, tW = pipe.profile(k=2)          # a1: the library's profiler (median, 1 us ticks)
    t_ref = sum(tF) // S
    host_c = max(gather(bench.measure_host_path(pipe, torch) if rank == 0 else 0))
    caps = {}
    for dd in gather({i: st.n_slots_fb for i, st in pipe.stages.items()}):
        caps.update(dd)
    x_cap = [caps[i] for i in range(S)]
    if any(a.endswith("-nccl") for a in args.arms.split(",")):
        pipe.enable_nccl(host_c)
    log = []

    n_iter = sy.PAPER_TRACE_ITERS // args.compress
    seq = []  # per iteration: (event id or -1, c, down)
    for k in range(n_iter):
        it = k * args.compress
        ev = next((e for e in sy.PAPER_TRACE if e["from"] <= it < e["to"]), None)
        if ev is None:
            seq.append((-1, [0] * (S - 1), []))
        else:
            c, down = bench.trace_c(ev, S, t_ref, host_c)
            seq.append((ev["id"], c, down))

    def run(name):
        base = Arm("adaptive" if name == "online" else name, S, N, tF, tB, tW, x_cap=x_cap, mem=(x_cap[0], 1))
        if name == "adaptive" and not log and rank == 0:
            log.append({"arm": name, "S": S, "N": N, "tF": tF, "tB": tB, "tW": tW, "x_cap": x_cap,
                        "mem": [x_cap[0], 1], "ratio": 30, "x_init": base.x_init})
        online = OnlinePlanner(base, t_ref) if name == "online" else None
        mon = LinkMonitor(pipe, gather)
        for l in range(S - 1):
            pipe.set_latency(l, 0)
        pipe.run(base.plan([0] * (S - 1)), merge_w=base.merge_w, inorder=base.inorder, nccl=base.nccl)  # warm-up
        mon.sample()
        if world > 1:
            dist.barrier(group=group)
        torch.cuda.synchronize()
        per_iter, busy_tot = [], 0
        for e, c, down in seq:
            for l in range(S - 1):
                want = L.LINK_DOWN if l in down else c[l]
                if pipe.latency[l] != want:
                    pipe.set_latency(l, want)
                pipe.set_path(l, base.deleg and c[l] > 0 and l not in down)
            orders = online.orders() if online else base.plan(c)
            if log and log[0]["arm"] == name and rank == 0:
                ent = dict(base.last)
                ent["step"] = len(per_iter)
                ent["orders"] = [" ".join(f"{kd}{mb}" for kd, mb in o) for o in orders]
                log.append(ent)
            ev0, ev1 = torch.cuda.Event(True), torch.cuda.Event(True)
            ev0.record()
            res = pipe.run(orders, merge_w=base.merge_w, inorder=base.inorder, nccl=base.nccl)
            if base.name == "adaptive":
                base.set_profile(*pipe.profile(k=5))
            ev1.record()
            torch.cuda.synchronize()
            g = gather((ev0.elapsed_time(ev1), sum(st["busy_ns"] for st in res.stats.values())))
            ms = max(v[0] for v in g)
            busy = sum(v[1] for v in g)
            busy_tot += busy
            per_iter.append((e, ms, 1 - busy / (S * ms * 1e6)))
            if online:
                meas, _ = mon.sample()
                online.observe(meas, down=down, host_c=host_c)
        tot = sum(x[1] for x in per_iter)
        return {"arm": name, "iterations": len(per_iter),
                "tokens_per_s": round(len(per_iter) * N * m.tokens_per_mb / (tot / 1e3), 1),
                "ms_per_iter": round(tot / len(per_iter), 2),
                "bubble": round(1 - busy_tot / (S * tot * 1e6), 4), "replans": base.replans,
                **({"nccl_probe_msgs": pipe.nccl_probe, "nccl_buffered": pipe.nccl_buffered} if base.nccl else {})}, per_iter

    out = {}
    for name in args.arms.split(","):
        out[name] = run(name)
    if args.replan_log and rank == 0:
        with open(args.replan_log, "w") as f:
            for e in log:
                f.write(json.dumps(e) + "\n")
    if rank == 0:
        meta = {"S": S, "N": N, "gpus": world, "layers": args.layers, "d": args.width,
                "compress": args.compress, "t_ref_us": t_ref / 1e3, "host_c_us": host_c / 1e3,
                "workload": f"C3 trace replay, {sy.PAPER_TRACE_ITERS} iterations compressed {args.compress}x"}
        for name, (summ, _) in out.items():
            summ.update(meta)
            print(json.dumps(summ), flush=True)
        for e in [-1] + [ev["id"] for ev in sy.PAPER_TRACE]:
            row = {"event": e if e >= 0 else "nominal"}
            if e >= 0:
                ev = sy.PAPER_TRACE[e]
                row.update({"links": ev["links"], "latency_ms_paper": ev["latency_ms"]})
            for name, (_, per_iter) in out.items():
                v = [x[1] for x in per_iter if x[0] == e]
                row[f"{name}_ms"] = round(sum(v) / len(v), 2) if v else None
                row[f"{name}_bubble"] = round(sum(x[2] for x in per_iter if x[0] == e) / len(v), 4) if v else None
            print(json.dumps(row), flush=True)
    pipe.close()
    if world > 1:
        dist.barrier(group=group)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
