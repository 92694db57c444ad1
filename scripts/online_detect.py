"""Online straggler detection study: the paper's trace replayed with
every event held for `--hold` iterations, on the same kernels and transport,
for three arms:
  informed  adaptive planner told the injected latencies (R18 lag 0 ablation)
  online    adaptive planner fed only the transport's measured per-message
            latencies, quantised with hysteresis, lag 1 (paper_2504_19232_b200.online)
  zb        fixed ZB order (Alg. 2 plan at c = 0)
One JSON line per arm (tokens/s, bubble, replans) plus a per-event detection
table (injected vs measured vs quantised latency) on rank 0.

  python scripts/online_detect.py [--S 4] [--N 16] [--layers 24] [--hold 4]
  (torchrun for several GPUs, as bench.py)
"""
import argparse
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--S", type=int, default=4)
    ap.add_argument("--N", type=int, default=16)
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--width", type=int, default=2048)
    ap.add_argument("--hold", type=int, default=4)
    ap.add_argument("--events", type=int, default=10)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import bench
    import synthetic as sy
    from paper_2504_19232_b200 import _lib as L
    from paper_2504_19232_b200 import sched as cs
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
    m = ModelCfg(block="gpt", n_layers=args.layers, d=args.width, d_ff=4 * args.width, n_heads=args.width // 128, b=1,
                 T=2048, dtype=L.BF16)
    pipe = Pipeline(m, S, N, rank=rank, world=world, device=local, group=group, host_links=True)
    prof = Arm("zb", S, N, [1000] * S, [1000] * S, [1000] * S)
    for _ in range(2):
        r = pipe.run(prof.orders)
    allp = {}
    for dd in gather({i: [st["op_ns"][k] // max(1, st["op_cnt"][k]) for k in range(3)] for i, st in r.stats.items()}):
        allp.update(dd)
    tF = [max(1, allp[i][0] // 1000) * 1000 for i in range(S)]
    tB = [max(1, allp[i][1] // 1000) * 1000 for i in range(S)]
    tW = [max(1, allp[i][2] // 1000) * 1000 for i in range(S)]
    t_ref = sum(tF) // S
    host_c = max(gather(bench.measure_host_path(pipe, torch) if rank == 0 else 0))
    caps = {}
    for dd in gather({i: st.n_slots_fb for i, st in pipe.stages.items()}):
        caps.update(dd)
    x_cap = [caps[i] for i in range(S)]
    x_init = cs.plan_init(S, N, x_cap[0], 1)
    x_init = [min(v, c) for v, c in zip(x_init, x_cap)]
    for i in range(S - 2, -1, -1):
        x_init[i] = max(x_init[i], x_init[i + 1])

    seq = []  # (event index, injected c, down links) per iteration
    for e, ev in enumerate(sy.PAPER_TRACE[:args.events]):
        c, down = bench.trace_c(ev, S, t_ref, host_c)
        seq += [(e, c, down)] * args.hold

    def run(name):
        base = Arm("zb" if name == "zb" else "adaptive", S, N, tF, tB, tW,
                   x_init=None if name == "zb" else x_init, x_cap=x_cap)
        online = OnlinePlanner(base, t_ref) if name == "online" else None
        mon = LinkMonitor(pipe, gather)
        for l in range(S - 1):
            pipe.set_latency(l, 0)
        pipe.run(base.plan([0] * (S - 1)), merge_w=False)  # warm-up at nominal
        mon.sample()
        if world > 1:
            dist.barrier(group=group)
        torch.cuda.synchronize()
        rows, tot_ms, busy_tot = [], 0.0, 0
        for e, c, down in seq:
            for l in range(S - 1):
                want = L.LINK_DOWN if l in down else c[l]
                if pipe.latency[l] != want:
                    pipe.set_latency(l, want)
            orders = online.orders() if online else base.plan(c)
            x_used = list(base.x)
            ev0, ev1 = torch.cuda.Event(True), torch.cuda.Event(True)
            ev0.record()
            res = pipe.run(orders, merge_w=False)
            ev1.record()
            torch.cuda.synchronize()
            g = gather((ev0.elapsed_time(ev1), sum(st["busy_ns"] for st in res.stats.values())))
            ms = max(v[0] for v in g)
            busy = sum(v[1] for v in g)
            meas, _mx = mon.sample()
            q = online.observe(meas, down=down, host_c=host_c) if online else None
            tot_ms += ms
            busy_tot += busy
            rows.append({"event": e, "injected_us": [v / 1e3 for v in c], "down": down,
                         "measured_us": [v / 1e3 for v in meas], "quantized_us": [v / 1e3 for v in q] if q else None,
                         "x": x_used, "ms": round(ms, 2), "bubble": round(1 - busy / (S * ms * 1e6), 4)})
        return {"arm": name, "iterations": len(seq), "tokens_per_s": round(len(seq) * N * m.tokens_per_mb / (tot_ms / 1e3), 1),
                "ms_per_iter": round(tot_ms / len(seq), 2), "bubble": round(1 - busy_tot / (S * tot_ms * 1e6), 4),
                "replans": base.replans}, rows

    out = {}
    for name in ("informed", "online", "zb"):
        out[name] = run(name)
    if rank == 0:
        for name, (summ, _) in out.items():
            summ.update({"S": S, "N": N, "gpus": world, "hold": args.hold, "t_ref_us": t_ref / 1e3,
                         "host_c_us": host_c / 1e3})
            print(json.dumps(summ), flush=True)
        # detection table: per event, mean measured / quantised on the straggling links (online arm)
        rows = out["online"][1]
        for e in sorted({r["event"] for r in rows}):
            er = [r for r in rows if r["event"] == e]
            print(json.dumps({"event": e, "injected_us": er[0]["injected_us"], "down": er[0]["down"],
                              "measured_us_first": er[0]["measured_us"], "measured_us_last": er[-1]["measured_us"],
                              "quantized_us_last": er[-1]["quantized_us"],
                              "x_first_iter": er[0]["x"], "x_last_iter": er[-1]["x"],
                              "ms_first_iter": er[0]["ms"], "ms_rest_mean": round(sum(r["ms"] for r in er[1:]) / max(1, len(er) - 1), 2),
                              "informed_ms_mean": round(sum(r["ms"] for r in out["informed"][1] if r["event"] == e) / len(er), 2)}),
                  flush=True)
    pipe.close()
    if world > 1:
        dist.barrier(group=group)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
