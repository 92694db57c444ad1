"""All-host-path overhead study (the paper's P:2616 analog: "< 5 %
overhead up to 30B, 17 % at 60B" with every inter-stage message delegated).

Same kernels, same adaptive planner, no stragglers; every link either on its
nominal NVLink path (DIRECT: the producer's epilogue writes the peer mailbox)
or forced onto the delegated path (D2H into the pinned shm ring on a side
stream, host flag, H2D by the receiver).  For the host arm the planner is
told every link costs the measured delegated-path latency (Alg. 2 re-plans
the warm-ups for it, as the paper does for a failed link).  One JSON line per
arm on rank 0, plus the measured one-message D2H+H2D time.

  python scripts/host_path_study.py [--S 4] [--N 16] [--layers 24] [--steps 5]
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
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import bench
    from paper_2504_19232_b200 import _lib as L
    from paper_2504_19232_b200 import sched as cs
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
    host_c = max(gather(bench.measure_host_path(pipe, torch) if rank == 0 else 0))
    caps = {}
    for dd in gather({i: st.n_slots_fb for i, st in pipe.stages.items()}):
        caps.update(dd)
    x_cap = [caps[i] for i in range(S)]
    x_init = cs.plan_init(S, N, x_cap[0], 1)
    x_init = [min(v, c) for v, c in zip(x_init, x_cap)]
    for i in range(S - 2, -1, -1):
        x_init[i] = max(x_init[i], x_init[i + 1])

    def run(host):
        arm = Arm("adaptive", S, N, tF, tB, tW, x_init=x_init, x_cap=x_cap)
        c = [host_c if host else 0] * (S - 1)
        for l in range(S - 1):
            pipe.set_latency(l, L.LINK_DOWN if host else 0)
        orders = arm.plan(c)
        pipe.run(orders)  # warm-up
        if world > 1:
            dist.barrier(group=group)
        torch.cuda.synchronize()
        tot, busy = 0.0, 0
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            res = pipe.run(orders)
            e1.record()
            torch.cuda.synchronize()
            g = gather((e0.elapsed_time(e1), sum(st["busy_ns"] for st in res.stats.values())))
            ms = max(v[0] for v in g)
            tot += ms
            busy += sum(v[1] for v in g)
        return {"arm": "all-host-path" if host else "nvlink", "x": arm.x,
                "tokens_per_s": round(args.steps * N * m.tokens_per_mb / (tot / 1e3), 1),
                "ms_per_iter": round(tot / args.steps, 2), "bubble": round(1 - busy / (S * tot * 1e6), 4)}

    res = [run(False), run(True)]
    for l in range(S - 1):
        pipe.set_latency(l, 0)
    if rank == 0:
        base = res[0]["tokens_per_s"]
        for r_ in res:
            r_.update({"S": S, "N": N, "gpus": world, "layers": args.layers, "d": args.width,
                       "msg_MiB": pipe.msg_bytes / 2**20, "host_path_us": host_c / 1e3,
                       "t_F_us": sum(tF) / S / 1e3, "overhead_vs_nvlink": round(1 - r_["tokens_per_s"] / base, 4)})
            print(json.dumps(r_), flush=True)
    pipe.close()
    if world > 1:
        dist.barrier(group=group)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
