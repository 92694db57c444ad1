"""Repeat the adaptive GPT pipeline iteration with injected latency many times
(flushes out intermittent transport races); prints any error verbatim."""
import os
import sys
import time

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("ADAPTRA_TIMEOUT_MS", "20000")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synthetic as sy  # noqa: E402
from paper_2504_19232_b200 import _lib as L  # noqa: E402
from paper_2504_19232_b200.pipeline import Arm, ModelCfg, Pipeline  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
S, N, Lt, d, dff, H, T = 2, 4, 4, 256, 1024, 2, 128
params = sy.gpt_params(0, S, Lt // S, d, dff, perturb=True, bf16=True)
xs = sy.microbatches(1, N, 1, T, d, bf16=True)
tg = sy.targets(2, N, 1, T, d)
m = ModelCfg(block="gpt", n_layers=Lt, d=d, d_ff=dff, n_heads=H, b=1, T=T, dtype=L.BF16)
fails = 0
for r in range(reps):
    pipe = Pipeline(m, S, N, params=params, inputs=xs, targets=tg)
    try:
        a = Arm("adaptive", S, N, [1000] * S, [1000] * S, [1000] * S)
        c = [2_000_000]
        pipe.set_latency(0, c[0])
        orders = a.plan(c)
        for it in range(3):
            t0 = time.time()
            res = pipe.run(orders, merge_w=a.merge_w)
        print(f"rep {r}: ok loss {res.loss:.5f} ({time.time() - t0:.3f}s)", flush=True)
    except Exception as e:
        fails += 1
        print(f"rep {r}: FAIL {e!r} orders={orders} links={pipe.link_stats()}", flush=True)
    finally:
        pipe.close()
print("fails", fails)
