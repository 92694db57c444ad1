"""NVLink evidence for the DIRECT link mode (a9): the stage's last GEMM
(FC2 + bias + residual, the F op's output) writes its epilogue straight into
the receiving stage's mailbox on the peer GPU.  Times that GEMM with C on the
local GPU and with C on GPU 1 (peer pointer, plain stores over NVLink), and
the output bytes per second that cross the link.  Run under ncu with
--metrics nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum for the
link byte counts.  Needs 2 GPUs (single process): gpurun --gpus 2."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_19232_b200 import _lib as L  # noqa: E402
from paper_2504_19232_b200 import ops  # noqa: E402

assert torch.cuda.device_count() >= 2, "needs 2 GPUs"
T, d = 2048, int(os.environ.get("D", 2048))
f = 4 * d
reps = int(os.environ.get("REPS", 20))
torch.cuda.set_device(0)
torch.cuda.set_device(1)
torch.cuda.set_device(0)
# enable peer access 0 -> 1 (the outbox does this for cross-GPU links)
torch.zeros(1, device="cuda:1")
try:
    torch.cuda.set_device(0)
    import ctypes
    cudart = ctypes.CDLL("libcudart.so")
    cudart.cudaDeviceEnablePeerAccess(1, 0)
except Exception:
    pass
g = torch.Generator(device="cuda:0").manual_seed(0)
A = (torch.randn(T, f, device="cuda:0", generator=g) * 0.1).to(torch.bfloat16)      # g (FC1 output)
W2 = (torch.randn(d, f, device="cuda:0", generator=g) * 0.02).to(torch.bfloat16)    # [out, in]
R = torch.randn(T, d, device="cuda:0", generator=g).to(torch.bfloat16)              # residual
bias = torch.zeros(d, device="cuda:0")
out = {}
for where in ("local", "peer"):
    C = torch.empty(T, d, device="cuda:0" if where == "local" else "cuda:1", dtype=torch.bfloat16)
    run = lambda: ops.gemm(A, W2, C, M=T, N=d, K=f, epi=L.EPI_RESID, R=R, bias=bias)
    for _ in range(3):
        run()
    torch.cuda.synchronize(0)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize(0)
    ms = e0.elapsed_time(e1) / reps
    out[where] = {"us": round(ms * 1e3, 1), "tflops": round(2 * T * d * f / ms / 1e9, 1),
                  "out_bytes": T * d * 2, "out_GBps": round(T * d * 2 / ms / 1e6, 1)}
    ref = C.to("cuda:0")
    out[where]["checksum"] = float(ref.float().abs().sum())
print(json.dumps({"gemm": "F_fc2 (FC2 + bias + residual), C1 shapes", **out,
                  "slowdown_peer_vs_local": round(out["peer"]["us"] / out["local"]["us"], 3),
                  "nvlink_peak_GBps": 900.0}), flush=True)
