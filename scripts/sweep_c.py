"""C4 sweep: tokens/s and bubble rate vs injected latency
c in {0, 1/4, 1/2, 1, 2, 4} x t_F on one link at a time (first, middle, last),
for the adaptive, fixed-ZB, fixed-1F1B and in-order (HOL) arms on the same
kernels.  One JSON line per (link, c, arm) on rank 0.

  python scripts/sweep_c.py [--model 1.3b|7b] [--S 4] [--N 16] [--steps 2]
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
    ap.add_argument("--model", default="1.3b", choices=["1.3b", "7b"])
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--S", type=int, default=4)
    ap.add_argument("--N", type=int, default=16)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--mults", default="0,0.25,0.5,1,2,4")
    ap.add_argument("--arms", default="adaptive,zb,1f1b,zb-inorder")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

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
    nl, d, h = (32, 4096, 32) if args.model == "7b" else (24, 2048, 16)
    nl = args.layers or nl
    S, N = args.S, args.N
    m = ModelCfg(block="gpt", n_layers=nl, d=d, d_ff=4 * d, n_heads=h, b=1, T=2048, dtype=L.BF16)
    pipe = Pipeline(m, S, N, rank=rank, world=world, device=local, group=group)

    def gather(o):
        if world == 1:
            return [o]
        out = [None] * world
        dist.all_gather_object(out, o, group=group)
        return out

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
    caps = {}
    for dd in gather({i: st.n_slots_fb for i, st in pipe.stages.items()}):
        caps.update(dd)
    x_cap = [caps[i] for i in range(S)]
    x_init = cs.plan_init(S, N, x_cap[0], 1)
    links = sorted({0, (S - 1) // 2, S - 2})
    for link in links:
        for mult in [float(v) for v in args.mults.split(",")]:
            c = [0] * (S - 1)
            c[link] = int(mult * t_ref)
            for l in range(S - 1):
                pipe.set_latency(l, c[l])
            for name in args.arms.split(","):
                arm = Arm(name, S, N, tF, tB, tW, x_init=x_init if name == "adaptive" else None, x_cap=x_cap)
                orders = arm.plan(c)
                pipe.run(orders, merge_w=arm.merge_w, inorder=arm.inorder)  # warm-up
                if world > 1:
                    dist.barrier(group=group)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record()
                busy = 0
                for _ in range(args.steps):
                    res = pipe.run(orders, merge_w=arm.merge_w, inorder=arm.inorder)
                    busy += sum(st["busy_ns"] for st in res.stats.values())
                e1.record()
                torch.cuda.synchronize()
                g = gather((e0.elapsed_time(e1), busy))
                ms = max(x[0] for x in g) / args.steps
                busy = sum(x[1] for x in g) / args.steps
                if rank == 0:
                    print(json.dumps({"model": args.model, "S": S, "N": N, "gpus": world, "link": link,
                                      "c_over_tF": mult, "c_us": c[link] / 1e3, "arm": name,
                                      "tokens_per_s": round(N * m.tokens_per_mb / (ms / 1e3), 1),
                                      "ms_per_step": round(ms, 2), "bubble": round(1 - busy / (S * ms * 1e6), 4),
                                      "x": arm.x}), flush=True)
    pipe.close()
    if world > 1:
        dist.barrier(group=group)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
