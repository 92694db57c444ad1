import os
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import faulthandler, os, sys, time
faulthandler.dump_traceback_later(40, exit=True)
os.environ["ADAPTRA_DEBUG"] = "1"
os.environ.setdefault("ADAPTRA_TIMEOUT_MS", "10000")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synthetic as sy
from paper_2504_19232_b200 import _lib as L
from paper_2504_19232_b200.pipeline import Arm, ModelCfg, Pipeline
S, N = int(sys.argv[1]), int(sys.argv[2])
params = sy.mlp_params(0, S, 1, 64, 64)
xs = sy.microbatches(1, N, 1, 32, 64); tg = sy.targets(2, N, 1, 32, 64)
m = ModelCfg(block="mlp", n_layers=S, d=64, d_ff=64, n_heads=1, b=1, T=32, dtype=L.F32)
pipe = Pipeline(m, S, N, params=params, inputs=xs, targets=tg, host_links=False)
print("built", flush=True)
a = Arm("1f1b", S, N, [1000] * S, [1000] * S, [1000] * S)
print("orders", a.orders, flush=True)
r = pipe.run(a.orders, merge_w=True)
print("ok loss", r.loss, flush=True)
pipe.close()
