"""Isolated timing of one stage's F / B / W ops (C1 layer shapes) with CUDA
events: NMB microbatches per op kind, REPS repetitions, the median per-op time
reported, plus the per-launch averages of the tcgen05 GEMM and the fused
attention kernels over the whole run.  OPB_W2=1 runs the W ops as W2 pairs
(K = 2bT).  Prints one JSON line."""
import ctypes
import json
import os
import statistics
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_19232_b200 import _lib as L  # noqa: E402
from paper_2504_19232_b200.stage import Stage  # noqa: E402

d, H, T, nl = int(os.environ.get("D", 2048)), 16, 2048, int(os.environ.get("LAYERS", 3))
nmb, reps = int(os.environ.get("NMB", 4)), int(os.environ.get("REPS", 8))
w2 = os.environ.get("OPB_W2") == "1"
wn = int(os.environ.get("OPB_WN", "0"))   # W of NMB slots in groups of wn (adaptra_stage_Wn)
st = Stage(L.BLOCK_GPT, L.BF16, nl, d, 4 * d, H, 1, T, False, False, nmb, nmb, "cuda")
g = torch.Generator(device="cuda").manual_seed(0)
st.wts.copy_((torch.randn(st.wts.numel(), device="cuda", generator=g) * 0.02).to(torch.bfloat16))
st.vecs.copy_(torch.ones(st.vecs.numel(), device="cuda"))
x = [torch.randn(T, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(nmb)]
y = [st.act() for _ in range(nmb)]
dy = [(torch.randn(T, d, device="cuda", generator=g) * 0.01).to(torch.bfloat16) for _ in range(nmb)]
dx = [st.act() for _ in range(nmb)]
times = {k: [] for k in "FBW"}
for rep in range(reps + 2):
    L.lib().adaptra_prof_enable(1 if rep >= 2 else 0)
    ev = {k: (torch.cuda.Event(True), torch.cuda.Event(True)) for k in "FBW"}
    ev["F"][0].record()
    for j in range(nmb):
        st.F(j, x[j], y[j])
    ev["F"][1].record()
    ev["B"][0].record()
    for j in range(nmb):
        st.B(j, dy[j], dx[j])
    ev["B"][1].record()
    ev["W"][0].record()
    if wn > 1:
        for j in range(0, nmb, wn):
            st.Wn(list(range(j, min(nmb, j + wn))))
    elif w2:
        for j in range(0, nmb - 1, 2):
            st.W2(j, j + 1)
        if nmb % 2:
            st.W(nmb - 1)
    else:
        for j in range(nmb):
            st.W(j)
    ev["W"][1].record()
    torch.cuda.synchronize()
    if rep >= 2:
        for k, e in ev.items():
            times[k].append(e[0].elapsed_time(e[1]) / nmb)
L.lib().adaptra_prof_enable(0)
res = {k: round(statistics.median(v), 4) for k, v in times.items()}
gf = 24 * T * d * d * nl / 1e9
af = 2 * T * T * d * nl / 1e9
res.update({"layers": nl, "nmb": nmb, "reps": reps, "w2": w2, "wn": wn,
            "env": {k: v for k, v in os.environ.items() if k.startswith("ADAPTRA_")},
            "F_tflops": round((gf + af) / res["F"] / 1e3, 1), "B_tflops": round((gf + 2 * af) / res["B"] / 1e3, 1),
            "W_tflops": round(gf / res["W"] / 1e3, 1)})
names = {0: "gemm_tc", 3: "attn_fwd", 4: "attn_bwd"}
for kind, nm in names.items():
    n, ms, fl, by = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    L.lib().adaptra_prof_collect(kind, n, ms, fl, by)
    if n.value:
        res[nm] = {"launches": n.value, "avg_us": round(ms.value * 1e3 / n.value, 2),
                   "tflops": round(fl.value / (ms.value / 1e3) / 1e12, 1)}
print(json.dumps(res), flush=True)
