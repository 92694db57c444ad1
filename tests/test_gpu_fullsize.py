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


@pytest.mark.parametrize("d,dff,H,nl,last", [
    (2048, 8192, 16, 1, False),     # C1 block
    (2048, 8192, 16, 1, True),      # C1 block, last stage (loss + dy seed)
    (2048, 8192, 16, 2, False),     # C1, two layers: 8 grouped dW products
    (4096, 16384, 32, 1, False),    # C2/C3 7B-shaped block
])
def test_full_size_block_fbw(d, dff, H, nl, last):
    T, b = 2048, 1
    params = sy.gpt_params(0, 1, nl, d, dff, perturb=True, bf16=True)[0]
    # scale the perturbed projections down to GPT-2 magnitudes at this width
    x = sy.microbatches(1, 1, b, T, d, bf16=True)[0]
    tgt = sy.targets(2, 1, b, T, d)[0]
    dy = sy.microbatches(3, 1, b, T, d, bf16=True)[0]
    st = Stage(L.BLOCK_GPT, L.BF16, nl, d, dff, H, b, T, False, last, 1, 1, "cuda")
    st.load_params(params)
    st.zero_grads()
    xin = torch.from_numpy(x.reshape(T, d)).to("cuda", torch.bfloat16)
    y = st.act()
    dx = st.act()
    loss = torch.zeros(1, device="cuda")
    st.F(0, xin, y, torch.from_numpy(tgt.reshape(T, d)).cuda() if last else None, loss if last else None)
    st.B(0, None if last else torch.from_numpy(dy.reshape(T, d)).to("cuda", torch.bfloat16), dx)
    st.W(0)
    torch.cuda.synchronize()
    p64 = [{k: np.asarray(v, np.float64) for k, v in layer.items()} for layer in params]
    yr, caches = nu.stage_F("gpt", p64, x.astype(np.float64), H)
    if last:
        Lr, dyr = nu.mse_loss(yr, tgt.astype(np.float64), 1)
        assert abs(loss.item() - Lr) <= 2e-2 * abs(Lr)
    else:
        dyr = dy.astype(np.float64)
        assert rel(y.double().cpu().numpy().reshape(yr.shape), yr) < 2e-2
    dxr, gc = nu.stage_B("gpt", p64, caches, dyr, H)
    assert rel(dx.double().cpu().numpy().reshape(dxr.shape), dxr) < 2e-2
    gw = nu.stage_W("gpt", caches, gc)
    got = st.grads()
    for l in range(nl):
        for k, ref in gw[l].items():
            e = rel(got[l][k], ref)
            assert e < 2e-2, (l, k, e)
