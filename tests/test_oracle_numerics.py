"""Pins for the numerics oracle (oracle/numerics.py): forward against independent
library routines (torch.nn.functional, float64), the F/B/W split against torch
autograd and central finite differences, closed-form invariants, and the exact
identity "pipelined B+W gradients == unpipelined full-batch gradients" (P12)."""
import numpy as np
import pytest
import torch
import torch.nn.functional as Fn

from oracle import numerics as nu
from oracle import sched as sc
import synthetic as sy


def _torch_block(kind, p, x, H):
    if kind == "mlp":
        return x + Fn.gelu(x @ p["W1"].T + p["b1"], approximate="tanh") @ p["W2"].T + p["b2"]
    d = x.shape[-1]
    b, T = x.shape[0], x.shape[1]
    h1 = Fn.layer_norm(x, (d,), p["ln1_g"], p["ln1_b"], 1e-5)
    qkv = h1 @ p["Wqkv"].T + p["bqkv"]
    q, k, v = [z.reshape(b, T, H, d // H).transpose(1, 2) for z in qkv.split(d, -1)]
    o = Fn.scaled_dot_product_attention(q, k, v, is_causal=True).transpose(1, 2).reshape(b, T, d)
    y1 = x + o @ p["Wo"].T + p["bo"]
    h2 = Fn.layer_norm(y1, (d,), p["ln2_g"], p["ln2_b"], 1e-5)
    return y1 + Fn.gelu(h2 @ p["W1"].T + p["b1"], approximate="tanh") @ p["W2"].T + p["b2"]


def _torch_loss_and_grads(kind, P, xs, tg, H):
    tp = [[{k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in blk.items()}
           for blk in st] for st in P]
    X = torch.tensor(np.concatenate(xs), dtype=torch.float64, requires_grad=True)
    Tg = torch.tensor(np.concatenate(tg), dtype=torch.float64)
    h = X
    for st in tp:
        for p in st:
            h = _torch_block(kind, p, h, H)
    L = 0.5 * ((h - Tg) ** 2).sum() / h.numel()
    L.backward()
    return L.item(), [[{k: v.grad.numpy() for k, v in blk.items()} for blk in st] for st in tp], X.grad.numpy()


CASES = [("mlp", 2, 2, 16, 24, None, 8, 1, 3), ("gpt", 2, 2, 32, 64, 2, 16, 1, 4),
         ("gpt", 3, 1, 24, 48, 3, 8, 2, 3)]


@pytest.mark.parametrize("kind,S,L,d,dff,H,T,b,N", CASES)
def test_forward_and_grads_vs_torch_autograd(kind, S, L, d, dff, H, T, b, N):
    P = sy.mlp_params(0, S, L, d, dff) if kind == "mlp" else sy.gpt_params(0, S, L, d, dff)
    xs = sy.microbatches(1, N, b, T, d)
    tg = sy.targets(2, N, b, T, d)
    Lt, gt, dxt = _torch_loss_and_grads(kind, P, xs, tg, H)
    L, g, dx = nu.full_batch(kind, P, xs, tg, H)
    assert abs(L - Lt) <= 1e-12 * abs(Lt)
    assert np.abs(dx - dxt).max() <= 1e-12 * np.abs(dxt).max()
    for i in range(S):
        for l in range(len(P[i])):
            for k in g[i][l]:
                ref = gt[i][l][k]
                assert np.abs(g[i][l][k] - ref).max() <= 1e-10 * max(np.abs(ref).max(), 1e-30), k


def test_finite_differences_gpt():
    """Central differences on the float64 loss pin every gradient formula to the
    forward definition independently of any library."""
    S, L, d, dff, H, T, b, N = 1, 1, 8, 16, 2, 5, 1, 2
    P = sy.gpt_params(3, S, L, d, dff)
    xs = sy.microbatches(4, N, b, T, d)
    tg = sy.targets(5, N, b, T, d)
    _, g, _ = nu.full_batch("gpt", P, xs, tg, H)
    rng = np.random.default_rng(0)
    eps = 1e-6
    for name in sy.GPT_NAMES:
        arr = P[0][0][name]
        for _ in range(3):
            idx = tuple(rng.integers(0, s) for s in arr.shape)
            P64 = [[{k: np.asarray(v, np.float64).copy() for k, v in blk.items()} for blk in st] for st in P]
            P64[0][0][name][idx] += eps
            Lp, _, _ = nu.full_batch("gpt", P64, xs, tg, H)
            P64[0][0][name][idx] -= 2 * eps
            Lm, _, _ = nu.full_batch("gpt", P64, xs, tg, H)
            fd = (Lp - Lm) / (2 * eps)
            an = g[0][0][name][idx]
            assert abs(fd - an) <= 1e-6 * max(abs(an), 1e-3), (name, idx, fd, an)


def test_gelu_values_and_ln_invariants():
    assert nu.gelu(np.array(0.0)) == 0.0
    # tanh-GeLU(1) = 0.5 (1 + tanh(sqrt(2/pi) 1.044715))
    assert abs(nu.gelu(np.array(1.0)) - 0.8411919906082768) < 1e-15
    assert abs(nu.gelu(np.array(10.0)) - 10.0) < 1e-12 and abs(nu.gelu(np.array(-10.0))) < 1e-12
    x = np.random.default_rng(0).normal(3, 2, (4, 7, 64))
    h, xhat, _ = nu.layernorm(x, np.ones(64), np.zeros(64))
    assert np.abs(h.mean(-1)).max() < 1e-12
    assert np.abs(h.var(-1) - 64 / 64 / (1 + 1e-5 / x.var(-1))).max() < 1e-9


def test_attention_causal_invariants():
    rng = np.random.default_rng(1)
    b, T, d, H = 2, 6, 8, 2
    q, k, v = (rng.normal(size=(b, T, d)) for _ in range(3))
    o, P = nu.attention_fwd(q, k, v, H)
    assert np.allclose(P.sum(-1), 1.0)
    assert np.all(np.triu(P[0, 0], 1) == 0.0)
    assert np.allclose(o[:, 0, :], v[:, 0, :])       # first token attends only to itself
    # identical keys -> uniform causal average of values
    o2, _ = nu.attention_fwd(q, np.zeros_like(k), v, H)
    ref = np.cumsum(v, axis=1) / np.arange(1, T + 1)[None, :, None]
    assert np.allclose(o2, ref)


def test_mse_seed():
    y = np.ones((1, 2, 3))
    L, dy = nu.mse_loss(y, y, 4)
    assert L == 0.0 and np.all(dy == 0)
    L, dy = nu.mse_loss(y, np.zeros_like(y), 4)
    assert L == 0.5 and np.allclose(dy, 1.0 / 24)


@pytest.mark.parametrize("kind", ["mlp", "gpt"])
@pytest.mark.parametrize("arm", ["1f1b", "zb", "adaptive"])
def test_p12_pipelined_equals_full_batch(kind, arm):
    """P12: the schedule changes when ops run, not what they compute."""
    S, L, d, dff, H, T, b, N = 3, 2, 16, 32, 2, 8, 1, 6
    P = sy.mlp_params(0, S, L, d, dff) if kind == "mlp" else sy.gpt_params(0, S, L, d, dff)
    xs = sy.microbatches(1, N, b, T, d)
    tg = sy.targets(2, N, b, T, d)
    t = [10] * S
    if arm == "1f1b":
        X, _, _ = sc.schedule_1f1b(S, N, t, t, t, 1)
        order = nu.merged_order(X)
    elif arm == "zb":
        X, _, _ = sc.schedule_zb(S, N, t, t, t, 1)
        order = nu.global_order(X)
    else:
        c = [0, 35]
        X, _, _ = sc.schedule(S, N, t, t, t, c, sc.get_adapted_warmup_fwds(S, N, t, t, c), 1)
        order = nu.global_order(X)
    for dtype, tol in ((np.float64, 1e-12), (np.float32, 1e-5)):
        Lp, gp, dxp = nu.pipeline_step(kind, P, xs, tg, order, H, dtype)
        Lf, gf, dxf = nu.full_batch(kind, P, xs, tg, H, dtype)
        assert abs(Lp - Lf) <= tol * abs(Lf)
        for i in range(S):
            for l in range(L):
                for k in gf[i][l]:
                    den = max(np.abs(gf[i][l][k]).max(), 1e-30)
                    assert np.abs(gp[i][l][k] - gf[i][l][k]).max() <= tol * den * 10, (k, dtype)
        dx_pipe = np.concatenate([dxp[j] for j in range(1, N + 1)])
        assert np.abs(dx_pipe - dxf).max() <= tol * np.abs(dxf).max() * 10
