"""Stage F / B / W through the C-ABI vs the float64 CPU oracle on the same
seeded inputs (north_star tolerances: max relative error 1e-4 fp32, 2e-2 bf16,
R20: max|g - g_ref| / max|g_ref| per tensor)."""
import numpy as np
import pytest
import torch

from oracle import numerics as nu
import synthetic as sy
from paper_2504_19232_b200 import _lib as L
from paper_2504_19232_b200.stage import Stage

pytestmark = pytest.mark.gpu

TOL = {L.F32: 1e-4, L.BF16: 2e-2}


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


CASES = [
    # kind, dtype, L, d, dff, H, b, T, n_mb
    ("mlp", L.F32, 2, 64, 64, None, 1, 32, 3),
    ("mlp", L.BF16, 2, 256, 512, None, 1, 256, 2),
    ("gpt", L.F32, 2, 128, 256, 2, 1, 64, 2),
    ("gpt", L.F32, 1, 256, 512, 2, 2, 128, 2),
    ("gpt", L.BF16, 2, 256, 1024, 2, 1, 256, 2),
    ("gpt", L.BF16, 1, 256, 512, 2, 2, 128, 2),
    # 3 sequences x 4 heads x 16 query blocks = 192 attention items on the
    # persistent forward grid (148 CTAs): CTAs with one and with two items
    ("gpt", L.BF16, 1, 512, 1024, 4, 3, 2048, 1),
]


# W of slot groups (adaptra_stage_W2 / _Wn: 2 slots, or all of them when
# there are 3+) on the cases with >= 2 microbatches
CASES_PAIRS = [c + (p,) for c in CASES for p in (False, True) if not (p and c[-1] < 2)]


@pytest.mark.parametrize("last", [False, True])
@pytest.mark.parametrize("kind,dtype,nl,d,dff,H,b,T,nmb,pairs", CASES_PAIRS)
def test_stage_fbw_vs_oracle(kind, dtype, nl, d, dff, H, b, T, nmb, pairs, last):
    bf = dtype == L.BF16
    params = (sy.mlp_params(0, 1, nl, d, dff, bf16=bf) if kind == "mlp"
              else sy.gpt_params(0, 1, nl, d, dff, perturb=True, bf16=bf))[0]
    xs = sy.microbatches(1, nmb, b, T, d, bf16=bf)
    tg = sy.targets(2, nmb, b, T, d)
    dys = sy.microbatches(3, nmb, b, T, d, bf16=bf)
    block = L.BLOCK_MLP if kind == "mlp" else L.BLOCK_GPT
    st = Stage(block, dtype, nl, d, dff, H or 1, b, T, is_first=False, is_last=last, n_microbatches=nmb,
               n_slots=nmb, device="cuda")
    st.load_params(params)
    st.zero_grads()
    tdt = st.tdt
    xin = [torch.from_numpy(x.reshape(b * T, d)).to("cuda", tdt) for x in xs]
    tgt = [torch.from_numpy(t.reshape(b * T, d)).cuda() for t in tg]
    dyin = [torch.from_numpy(v.reshape(b * T, d)).to("cuda", tdt) for v in dys]
    ys = [st.act() for _ in range(nmb)]
    dxs = [st.act() for _ in range(nmb)]
    loss = torch.zeros(1, device="cuda")
    for j in range(nmb):
        st.F(j, xin[j], ys[j], tgt[j] if last else None, loss if last else None)
    for j in range(nmb):
        st.B(j, None if last else dyin[j], dxs[j])
        if not pairs:
            st.W(j)
    if pairs and nmb >= 3:      # all slots in one K = nmb bT launch
        st.Wn(list(range(nmb)))
    elif pairs:                 # W of slots (0,1), (2,3), ... as K = 2bT launches
        for j in range(0, nmb - 1, 2):
            st.W2(j, j + 1)
        if nmb % 2:
            st.W(nmb - 1)
    torch.cuda.synchronize()
    # oracle
    tol = TOL[dtype]
    gsum = None
    Lref = 0.0
    for j in range(nmb):
        x = xs[j].astype(np.float64)
        y, caches = nu.stage_F(kind, [dict(p) for p in params_list(params, nl)], x, H)
        if last:
            Lj, dy = nu.mse_loss(y, tg[j].astype(np.float64), nmb)
            Lref += Lj / nmb
        else:
            dy = dys[j].astype(np.float64)
            assert rel(ys[j].double().cpu().numpy().reshape(y.shape), y) < tol
        dx, gc = nu.stage_B(kind, params_list(params, nl), caches, dy, H)
        assert rel(dxs[j].double().cpu().numpy().reshape(dx.shape), dx) < tol
        gw = nu.stage_W(kind, caches, gc)
        if gsum is None:
            gsum = gw
        else:
            for l in range(nl):
                for k in gw[l]:
                    gsum[l][k] = gsum[l][k] + gw[l][k]
    if last:
        assert abs(loss.item() - Lref) <= tol * abs(Lref)
    got = st.grads()
    for l in range(nl):
        for k in gsum[l]:
            assert rel(got[l][k], gsum[l][k]) < tol, (l, k, rel(got[l][k], gsum[l][k]))


def params_list(stage_params, nl):
    return [{k: np.asarray(v, np.float64) for k, v in p.items()} for p in stage_params]
