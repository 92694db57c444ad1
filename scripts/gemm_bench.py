"""Time the tcgen05 GEMM on the C1 stage shapes (F, dX, dW layouts) with CUDA
events vs torch.matmul (cuBLAS) on identical shapes; prints one JSON per shape."""
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_19232_b200 import _lib as L  # noqa: E402
from paper_2504_19232_b200 import ops  # noqa: E402

T, d, f = 2048, int(os.environ.get("D", 2048)), 4 * int(os.environ.get("D", 2048))
reps = int(os.environ.get("REPS", 20))
shapes = [
    # name, M, N, K, a_mn, b_mn, epi
    ("F_qkv", T, 3 * d, d, 0, 0, L.EPI_STORE),
    ("F_o", T, d, d, 0, 0, L.EPI_RESID),
    ("F_o_plain", T, d, d, 0, 0, L.EPI_STORE),
    ("F_fc1", T, f, d, 0, 0, L.EPI_GELU),
    ("F_fc2", T, d, f, 0, 0, L.EPI_RESID),
    ("B_fc2", T, f, d, 0, 1, L.EPI_DGELU),
    ("B_fc1", T, d, f, 0, 1, L.EPI_STORE),
    ("B_qkv", T, d, 3 * d, 0, 1, L.EPI_STORE),
    ("W_fc2", d, f, T, 1, 1, L.EPI_ACC_F32),
    ("W_fc1", f, d, T, 1, 1, L.EPI_ACC_F32),
    ("W_qkv", 3 * d, d, T, 1, 1, L.EPI_ACC_F32),
]
only = os.environ.get("ONLY")
dev = "cuda"
for name, M, N, K, amn, bmn, epi in shapes:
    if only and only not in name:
        continue
    A = (torch.randn(K, M) if amn else torch.randn(M, K)).to(dev, torch.bfloat16)
    B = (torch.randn(K, N) if bmn else torch.randn(N, K)).to(dev, torch.bfloat16)
    f32 = epi == L.EPI_ACC_F32
    Cm = torch.zeros(M, N, device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
    kw = {}
    if epi in (L.EPI_GELU, L.EPI_DGELU):
        kw["aux"] = torch.randn(M, N, device=dev).to(torch.bfloat16)
    if epi == L.EPI_RESID:
        kw["R"] = torch.randn(M, N, device=dev).to(torch.bfloat16)
    if epi in (L.EPI_GELU, L.EPI_RESID, L.EPI_STORE) and not name.endswith("_plain"):
        kw["bias"] = torch.randn(N, device=dev)
    run = lambda: ops.gemm(A, B, Cm, M=M, N=N, K=K, a_mn=amn, b_mn=bmn, epi=epi, **kw)
    Am = A.t() if amn else A
    Bm = B.t() if bmn else B
    ref = lambda: torch.matmul(Am, Bm.t())
    for fn in (run, ref):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    res = {}
    for tag, fn in (("ours", run), ("cublas", ref)):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[tag] = {"us": round(ms * 1e3, 1), "tflops": round(2 * M * N * K / ms / 1e9, 1)}
    print(json.dumps({"shape": name, "M": M, "N": N, "K": K, **res}), flush=True)
