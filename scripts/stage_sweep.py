"""Config C4: stage-count x microbatch sweep on the same
kernels, GPT blocks of the 1.3B-shaped stack (24 layers, d = 2048, T = 2048),
S in {2, 4, 8} and N in {8, 32, 64} (combinations whose stash fits the
devices), for the adaptive, fixed ZB and fixed 1F1B arms, without stragglers
and with c = 2 t_F on the middle link.  N = 8 with S = 8 exercises the N < 2S
clamp of Alg. 2 (R11).  Stages map to GPUs contiguously (stage i on GPU
i * world // S).  One JSON line per (S, N, arm, condition) on rank 0.

  python -m torch.distributed.run --nproc-per-node 4 ... scripts/stage_sweep.py
"""
import argparse
import gc
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ["NCCL_DEBUG"] = "WARN"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2x8,2x32,4x8,4x32,4x64,8x8,8x32,8x64")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--mult", type=float, default=2.0)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_2504_19232_b200 import _lib as L
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

    m = ModelCfg(block="gpt", n_layers=24, d=2048, d_ff=8192, n_heads=16, b=1, T=2048, dtype=L.BF16)
    for cfg in args.configs.split(","):
        S, N = (int(v) for v in cfg.split("x"))
        pipe = Pipeline(m, S, N, rank=rank, world=world, device=local, group=group, host_links=True)
        # a1 as in bench.py: the library profiler (median of the last
        # iterations, 1 us ticks) on the ZB order at c = 0; Alg. 1's memory
        # input and the R26 clamp from each stage's F->B stash capacity
        prof = Arm("zb", S, N, [1000] * S, [1000] * S, [1000] * S)
        for _ in range(3):
            pipe.run(prof.orders)
        tF, tB, tW = pipe.profile(k=2)
        t_ref = sum(tF) // S
        caps = {}
        for dd in gather({i: st.n_slots_fb for i, st in pipe.stages.items()}):
            caps.update(dd)
        x_cap = [caps[i] for i in range(S)]
        for cond in ("nominal", "straggler"):
            c = [0] * (S - 1)
            if cond == "straggler":
                c[(S - 1) // 2] = int(args.mult * t_ref)
            for l in range(S - 1):
                pipe.set_latency(l, c[l])
            for name in ("adaptive", "zb", "1f1b"):
                arm = Arm(name, S, N, tF, tB, tW, x_cap=x_cap, mem=(x_cap[0], 1))
                orders = arm.plan(c)
                pipe.run(orders, merge_w=arm.merge_w)
                if world > 1:
                    dist.barrier(group=group)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record()
                busy = 0
                for _ in range(args.steps):
                    res = pipe.run(orders, merge_w=arm.merge_w)
                    busy += sum(st["busy_ns"] for st in res.stats.values())
                e1.record()
                torch.cuda.synchronize()
                g = gather((e0.elapsed_time(e1), busy))
                ms = max(v[0] for v in g) / args.steps
                busy = sum(v[1] for v in g) / args.steps
                if rank == 0:
                    print(json.dumps({"S": S, "N": N, "gpus": world, "stage_map": [i * world // S for i in range(S)],
                                      "condition": cond, "c_over_tF": args.mult if cond == "straggler" else 0,
                                      "arm": name, "x": arm.x, "tokens_per_s": round(N * m.tokens_per_mb / (ms / 1e3), 1),
                                      "ms_per_step": round(ms, 2), "bubble": round(1 - busy / (S * ms * 1e6), 4)}),
                          flush=True)
        for l in range(S - 1):
            pipe.set_latency(l, 0)
        pipe.close()
        del pipe
        gc.collect()
        torch.cuda.empty_cache()
        if world > 1:
            dist.barrier(group=group)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
