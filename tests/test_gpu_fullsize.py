"""Parity at BASELINE.json's full sizes: GPT-2 blocks of the 1.3B-shaped stack
(C1: d=2048, 16 heads x 128, d_ff=8192) and of the 7B-shaped stack (C2/C3:
d=4096, 32 heads x 128, d_ff=16384), T=2048 tokens, bf16, run through the same
C-ABI stage calls and kernel configurations as bench.py (2-CTA 256x256
tcgen05 tiles, fused flash attention, the grouped dW launch: 4 products per
layer, 8 with two layers) against the float64 oracle on the same inputs:
every element of y, dx and every gradient, tolerance 2e-2 (max relative
error, R20)."""
import numpy as np
import pytest
import torch

from oracle import numerics as nu
import synthetic as sy
from paper_2504_19232_b200 import _lib as L
from paper_2504_19232_b200.stage import Stage

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.mark.parametrize("d,dff,H,nl,last,nmb", [
    (2048, 8192, 16, 1, False, 1),     # C1 block
    (2048, 8192, 16, 1, True, 1),      # C1 block, last stage (loss + dy seed)
    (2048, 8192, 16, 2, False, 1),     # C1, two layers: 8 grouped dW products
    (4096, 16384, 32, 1, False, 1),    # C2/C3 7B-shaped block
    (2048, 8192, 16, 1, False, 2),     # C1, W of two slots in one launch (K = 2bT, stage_Wn)
])
def test_full_size_block_fbw(d, dff, H, nl, last, nmb):
    """Every gradient of the W op at C1 / 7B sizes, including the bias
    gradients the grouped dW launch sums from its staged dY tiles."""
    T, b = 2048, 1
    params = sy.gpt_params(0, 1, nl, d, dff, perturb=True, bf16=True)[0]
    xs = sy.microbatches(1, nmb, b, T, d, bf16=True)
    tgs = sy.targets(2, nmb, b, T, d)
    dys = sy.microbatches(3, nmb, b, T, d, bf16=True)
    st = Stage(L.BLOCK_GPT, L.BF16, nl, d, dff, H, b, T, False, last, nmb, nmb, "cuda")
    st.load_params(params)
    st.zero_grads()
    ys = [st.act() for _ in range(nmb)]
    dxs = [st.act() for _ in range(nmb)]
    loss = torch.zeros(1, device="cuda")
    # W reads the F input and the B input gradient in place (the mailbox
    # contract): they stay alive until W
    xin = [torch.from_numpy(x.reshape(T, d)).to("cuda", torch.bfloat16) for x in xs]
    dyin = [torch.from_numpy(v.reshape(T, d)).to("cuda", torch.bfloat16) for v in dys]
    tgin = [torch.from_numpy(t.reshape(T, d)).cuda() for t in tgs]
    for j in range(nmb):
        st.F(j, xin[j], ys[j], tgin[j] if last else None, loss if last else None)
    for j in range(nmb):
        st.B(j, None if last else dyin[j], dxs[j])
    if nmb == 1:
        st.W(0)
    else:
        st.Wn(list(range(nmb)))
    torch.cuda.synchronize()
    p64 = [{k: np.asarray(v, np.float64) for k, v in layer.items()} for layer in params]
    gsum, Lr = None, 0.0
    for j in range(nmb):
        yr, caches = nu.stage_F("gpt", p64, xs[j].astype(np.float64), H)
        if last:
            Lj, dyr = nu.mse_loss(yr, tgs[j].astype(np.float64), nmb)
            Lr += Lj / nmb
        else:
            dyr = dys[j].astype(np.float64)
            assert rel(ys[j].double().cpu().numpy().reshape(yr.shape), yr) < 2e-2
        dxr, gc = nu.stage_B("gpt", p64, caches, dyr, H)
        assert rel(dxs[j].double().cpu().numpy().reshape(dxr.shape), dxr) < 2e-2
        gw = nu.stage_W("gpt", caches, gc)
        gsum = gw if gsum is None else [{k: gsum[l][k] + gw[l][k] for k in gw[l]} for l in range(nl)]
    if last:
        assert abs(loss.item() - Lr) <= 2e-2 * abs(Lr)
    got = st.grads()
    errs = {(l, k): rel(got[l][k], ref) for l in range(nl) for k, ref in gsum[l].items()}
    assert max(errs.values()) < 2e-2, errs
