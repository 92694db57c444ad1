"""Isolated timing of one stage's F / B / W ops (C1 layer shapes) with CUDA events."""
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_19232_b200 import _lib as L  # noqa: E402
from paper_2504_19232_b200.stage import Stage  # noqa: E402

d, H, T, nl = int(os.environ.get("D", 2048)), 16, 2048, int(os.environ.get("LAYERS", 6))
st = Stage(L.BLOCK_GPT, L.BF16, nl, d, 4 * d, H, 1, T, False, False, 4, 4, "cuda")
g = torch.Generator(device="cuda").manual_seed(0)
st.wts.copy_((torch.randn(st.wts.numel(), device="cuda", generator=g) * 0.02).to(torch.bfloat16))
v = torch.zeros(st.vecs.numel(), device="cuda")
st.vecs.copy_(v + 1.0)
x = [torch.randn(T, d, device="cuda").to(torch.bfloat16) for _ in range(4)]
y = [st.act() for _ in range(4)]
dy = [torch.randn(T, d, device="cuda").to(torch.bfloat16) * 0.01 for _ in range(4)]
dx = [st.act() for _ in range(4)]
import ctypes  # noqa: E402

res = {}
for rep in range(3):
    L.lib().adaptra_prof_enable(1 if rep == 2 else 0)
    ev = {k: (torch.cuda.Event(True), torch.cuda.Event(True)) for k in "FBW"}
    ev["F"][0].record()
    for j in range(4):
        st.F(j, x[j], y[j])
    ev["F"][1].record()
    ev["B"][0].record()
    for j in range(4):
        st.B(j, dy[j], dx[j])
    ev["B"][1].record()
    ev["W"][0].record()
    for j in range(4):
        st.W(j)
    ev["W"][1].record()
    torch.cuda.synchronize()
    res = {k: round(e[0].elapsed_time(e[1]) / 4, 3) for k, e in ev.items()}
gf = 24 * T * d * d * nl / 1e9
af = 2 * T * T * d * nl / 1e9
res.update({"layers": nl, "attn": os.environ.get("ADAPTRA_ATTN", "fused"),
            "F_tflops": round((gf + af) / res["F"] / 1e3, 1), "B_tflops": round((gf + 2 * af) / res["B"] / 1e3, 1),
            "W_tflops": round(gf / res["W"] / 1e3, 1)})
L.lib().adaptra_prof_enable(0)
names = {0: "gemm_tc", 2: "gemm_attn", 3: "attn_fwd", 4: "attn_bwd"}
for kind, nm in names.items():
    n, ms, fl, by = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    L.lib().adaptra_prof_collect(kind, n, ms, fl, by)
    if n.value:
        res[nm] = {"launches": n.value, "avg_us": round(ms.value * 1e3 / n.value, 2),
                   "tflops": round(fl.value / (ms.value / 1e3) / 1e12, 1)}
print(json.dumps(res))
