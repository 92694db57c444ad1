"""Debug: smallest pipelines, printing progress (run on the GPU box)."""
import os
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import faulthandler
import os
import sys
import time

faulthandler.dump_traceback_later(100, exit=True)
os.environ.setdefault("ADAPTRA_TIMEOUT_MS", "15000")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synthetic as sy  # noqa: E402
from paper_2504_19232_b200 import _lib as L  # noqa: E402
from paper_2504_19232_b200.pipeline import Arm, ModelCfg, Pipeline  # noqa: E402

for S, N, mode in ((2, 2, L.LINK_DIRECT), (4, 8, L.LINK_DIRECT), (4, 8, L.LINK_P2P)):
    params = sy.mlp_params(0, S, 1, 64, 64)
    xs = sy.microbatches(1, N, 1, 32, 64)
    tg = sy.targets(2, N, 1, 32, 64)
    m = ModelCfg(block="mlp", n_layers=S, d=64, d_ff=64, n_heads=1, b=1, T=32, dtype=L.F32)
    t0 = time.time()
    pipe = Pipeline(m, S, N, params=params, inputs=xs, targets=tg, link_mode=mode)
    print("built", S, N, mode, time.time() - t0, flush=True)
    for arm in ("1f1b", "zb"):
        a = Arm(arm, S, N, [1000] * S, [1000] * S, [1000] * S)
        try:
            r = pipe.run(a.orders, merge_w=a.merge_w)
            print(arm, "ok loss", r.loss, {i: s["busy_ns"] for i, s in r.stats.items()}, flush=True)
        except Exception as e:
            print(arm, "FAILED", e, flush=True)
    pipe.set_latency(0, 3_000_000)
    a = Arm("zb", S, N, [1000] * S, [1000] * S, [1000] * S)
    try:
        r = pipe.run(a.orders, want_times=True)
        print("lat ok", r.stats[0]["op_times"][:3], r.stats[1]["op_times"][:3], flush=True)
    except Exception as e:
        print("lat FAILED", e, flush=True)
    pipe.set_latency(0, L.LINK_DOWN)
    try:
        r = pipe.run(a.orders)
        print("down ok loss", r.loss, flush=True)
    except Exception as e:
        print("down FAILED", e, flush=True)
    pipe.close()
print("done")
