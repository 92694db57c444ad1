"""CPU oracle for the numerical content of one zero-bubble pipeline step.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may use it; the CUDA
path never imports it and shares no code with it.

Plain numpy, float64 by default (float32 on request), hand-written forward and
backward, no autograd.  What it computes:

* per stage, L_s identical blocks; a microbatch is a tensor x[b, T, d] of whole
  sequences (b sequences of T tokens);
* block "mlp" (config C0, reading R24): y = x + gelu(x W1^T + b1) W2^T + b2;
* block "gpt" (GPT-2 pre-LN block, "GPT-2"): LN1 -> QKV -> causal
  multi-head attention -> O (+residual) -> LN2 -> FC1 -> GeLU -> FC2 (+residual);
* gelu is GPT-2's tanh form (reading R25); LayerNorm eps = 1e-5;
* loss (R19): L_j = (1/(b T d)) sum 1/2 (y - tgt)^2 per microbatch,
  L = (1/N) sum_j L_j, so dy seed = (y - tgt) / (N b T d);
* the backward is split as in ZeroBubble: B computes the input
  gradient only and keeps every GEMM's output gradient; W computes the weight
  gradients dW = dY^T X, db = sum dY (and LayerNorm dgamma, dbeta) later,
  accumulating across microbatches (deferred).

Weights use the [out, in] layout: a linear layer is y = x @ W.T + b.

Pins (tests/test_oracle_numerics.py): forward against torch.nn.functional in
float64 (layer_norm, gelu(approximate='tanh'), scaled_dot_product_attention
with is_causal), B+W against torch autograd and central finite differences,
LN/attention invariants, and pipelined B/W accumulation == full-batch gradient.
"""
from __future__ import annotations

import numpy as np

LN_EPS = 1e-5
_K0 = np.sqrt(2.0 / np.pi)
_K1 = 0.044715


def gelu(a):
    """GPT-2 tanh GeLU: 0.5 a (1 + tanh(sqrt(2/pi) (a + 0.044715 a^3)))."""
    return 0.5 * a * (1.0 + np.tanh(_K0 * (a + _K1 * a ** 3)))


def gelu_grad(a):
    """d gelu / d a for the tanh form."""
    u = _K0 * (a + _K1 * a ** 3)
    th = np.tanh(u)
    return 0.5 * (1.0 + th) + 0.5 * a * (1.0 - th ** 2) * _K0 * (1.0 + 3.0 * _K1 * a ** 2)


def linear(x, Wt, b):
    """y = x W^T + b over the last axis; W is [out, in]."""
    return x @ Wt.T + b


def layernorm(x, gamma, beta):
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + LN_EPS)
    xhat = (x - mu) * rstd
    return xhat * gamma + beta, xhat, rstd


def layernorm_bwd_x(dh, xhat, rstd, gamma):
    """dx for h = gamma * xhat + beta, xhat = (x - mean) * rstd."""
    g = dh * gamma
    return rstd * (g - g.mean(axis=-1, keepdims=True)
                   - xhat * (g * xhat).mean(axis=-1, keepdims=True))


def _heads(t, H):
    b, T, d = t.shape
    return t.reshape(b, T, H, d // H).transpose(0, 2, 1, 3)      # [b, H, T, dh]


def _merge(t):
    b, H, T, dh = t.shape
    return t.transpose(0, 2, 1, 3).reshape(b, T, H * dh)


def attention_fwd(q, k, v, H):
    """Causal softmax(q k^T / sqrt(dh)) v per head (plain definition)."""
    qh, kh, vh = _heads(q, H), _heads(k, H), _heads(v, H)
    T = q.shape[1]
    dh = q.shape[2] // H
    s = (qh @ kh.transpose(0, 1, 3, 2)) / np.sqrt(dh)
    mask = np.triu(np.ones((T, T), dtype=bool), k=1)             # key j > query i
    s = np.where(mask, -np.inf, s)
    s = s - s.max(axis=-1, keepdims=True)
    p = np.exp(s)
    p = p / p.sum(axis=-1, keepdims=True)
    o = p @ vh
    return _merge(o), p


def attention_bwd(do, q, k, v, p, H):
    qh, kh, vh = _heads(q, H), _heads(k, H), _heads(v, H)
    doh = _heads(do, H)
    dh_ = q.shape[2] // H
    dp = doh @ vh.transpose(0, 1, 3, 2)
    dv = p.transpose(0, 1, 3, 2) @ doh
    ds = p * (dp - (dp * p).sum(axis=-1, keepdims=True))
    scale = 1.0 / np.sqrt(dh_)
    dq = (ds @ kh) * scale
    dk = (ds.transpose(0, 1, 3, 2) @ qh) * scale
    return _merge(dq), _merge(dk), _merge(dv)


# ---------------------------------------------------------------------------
# Blocks: F / B / W
# ---------------------------------------------------------------------------

MLP_PARAMS = ("W1", "b1", "W2", "b2")
GPT_PARAMS = ("ln1_g", "ln1_b", "Wqkv", "bqkv", "Wo", "bo",
              "ln2_g", "ln2_b", "W1", "b1", "W2", "b2")


def block_F(kind, p, x, H=None):
    """Forward of one block. Returns (y, cache)."""
    if kind == "mlp":
        a = linear(x, p["W1"], p["b1"])
        g = gelu(a)
        y = x + linear(g, p["W2"], p["b2"])
        return y, {"x": x, "a": a, "g": g}
    h1, xhat1, rstd1 = layernorm(x, p["ln1_g"], p["ln1_b"])
    qkv = linear(h1, p["Wqkv"], p["bqkv"])
    d = x.shape[-1]
    q, k, v = qkv[..., :d], qkv[..., d:2 * d], qkv[..., 2 * d:]
    o, P = attention_fwd(q, k, v, H)
    y1 = x + linear(o, p["Wo"], p["bo"])
    h2, xhat2, rstd2 = layernorm(y1, p["ln2_g"], p["ln2_b"])
    a = linear(h2, p["W1"], p["b1"])
    g = gelu(a)
    y = y1 + linear(g, p["W2"], p["b2"])
    cache = {"h1": h1, "xhat1": xhat1, "rstd1": rstd1, "q": q, "k": k, "v": v,
             "P": P, "o": o, "h2": h2, "xhat2": xhat2, "rstd2": rstd2, "a": a, "g": g}
    return y, cache


def block_B(kind, p, cache, dy, H=None):
    """Input-gradient backward (ZB "B"). Returns (dx, gcache) where gcache holds
    each GEMM's output gradient (and LN output gradients) for W."""
    if kind == "mlp":
        dg = dy @ p["W2"]
        da = dg * gelu_grad(cache["a"])
        dx = dy + da @ p["W1"]
        return dx, {"dy": dy, "da": da}
    dg = dy @ p["W2"]
    da = dg * gelu_grad(cache["a"])
    dh2 = da @ p["W1"]
    dy1 = dy + layernorm_bwd_x(dh2, cache["xhat2"], cache["rstd2"], p["ln2_g"])
    do = dy1 @ p["Wo"]
    dq, dk, dv = attention_bwd(do, cache["q"], cache["k"], cache["v"], cache["P"], H)
    dqkv = np.concatenate([dq, dk, dv], axis=-1)
    dh1 = dqkv @ p["Wqkv"]
    dx = dy1 + layernorm_bwd_x(dh1, cache["xhat1"], cache["rstd1"], p["ln1_g"])
    return dx, {"dy": dy, "da": da, "dh2": dh2, "dy1": dy1, "dqkv": dqkv, "dh1": dh1}


def _wgrad(dY, X):
    """dW = dY^T X summed over all leading (token) axes; [out, in]."""
    return dY.reshape(-1, dY.shape[-1]).T @ X.reshape(-1, X.shape[-1])


def _bgrad(dY):
    return dY.reshape(-1, dY.shape[-1]).sum(axis=0)


def block_W(kind, cache, gcache):
    """Weight-gradient backward (ZB "W"). Returns dict of parameter gradients."""
    if kind == "mlp":
        return {"W1": _wgrad(gcache["da"], cache["x"]), "b1": _bgrad(gcache["da"]),
                "W2": _wgrad(gcache["dy"], cache["g"]), "b2": _bgrad(gcache["dy"])}
    return {
        "W2": _wgrad(gcache["dy"], cache["g"]), "b2": _bgrad(gcache["dy"]),
        "W1": _wgrad(gcache["da"], cache["h2"]), "b1": _bgrad(gcache["da"]),
        "ln2_g": _bgrad(gcache["dh2"] * cache["xhat2"]), "ln2_b": _bgrad(gcache["dh2"]),
        "Wo": _wgrad(gcache["dy1"], cache["o"]), "bo": _bgrad(gcache["dy1"]),
        "Wqkv": _wgrad(gcache["dqkv"], cache["h1"]), "bqkv": _bgrad(gcache["dqkv"]),
        "ln1_g": _bgrad(gcache["dh1"] * cache["xhat1"]), "ln1_b": _bgrad(gcache["dh1"]),
    }


def mse_loss(y, tgt, N):
    """R19: L_j = (1/(bTd)) sum 1/2 (y - tgt)^2; seed dy = (y - tgt)/(N b T d)."""
    n = y.size
    L = 0.5 * ((y - tgt) ** 2).sum() / n
    dy = (y - tgt) / (N * n)
    return L, dy


# ---------------------------------------------------------------------------
# Stages and the pipelined step
# ---------------------------------------------------------------------------

def _cast(params, dtype):
    return [[{k: np.asarray(v, dtype=dtype) for k, v in blk.items()} for blk in st] for st in params]


def stage_F(kind, stage_params, x, H=None):
    caches = []
    for p in stage_params:
        x, cch = block_F(kind, p, x, H)
        caches.append(cch)
    return x, caches


def stage_B(kind, stage_params, caches, dy, H=None):
    gcaches = [None] * len(stage_params)
    for l in range(len(stage_params) - 1, -1, -1):
        dy, gcaches[l] = block_B(kind, stage_params[l], caches[l], dy, H)
    return dy, gcaches


def stage_W(kind, caches, gcaches):
    return [block_W(kind, c, g) for c, g in zip(caches, gcaches)]


def zero_grads(params, dtype):
    return [[{k: np.zeros_like(np.asarray(v, dtype=dtype)) for k, v in blk.items()} for blk in st]
            for st in params]


def pipeline_step(kind, params, xs, tgts, order, H=None, dtype=np.float64):
    """Run one pipelined iteration in the global op order ``order`` = list of
    (stage, kind, mb) (mb 1-based), as a schedule would execute it: F caches
    activations, B caches output gradients, W accumulates weight gradients in
    the order W ops run (deferred accumulation).  Returns (loss, grads, dx0s)."""
    params = _cast(params, dtype)
    S = len(params)
    N = len(xs)
    grads = zero_grads(params, dtype)
    act_in = {(0, j): np.asarray(xs[j - 1], dtype=dtype) for j in range(1, N + 1)}
    caches, gcaches, grad_in = {}, {}, {}
    loss = 0.0
    dx0 = {}
    for (i, k, j) in order:
        if k == "F":
            y, caches[(i, j)] = stage_F(kind, params[i], act_in.pop((i, j)), H)
            if i == S - 1:
                Lj, dy = mse_loss(y, np.asarray(tgts[j - 1], dtype=dtype), N)
                loss += Lj / N
                grad_in[(i, j)] = dy
            else:
                act_in[(i + 1, j)] = y
        elif k == "B":
            dx, gcaches[(i, j)] = stage_B(kind, params[i], caches[(i, j)], grad_in.pop((i, j)), H)
            if i > 0:
                grad_in[(i - 1, j)] = dx
            else:
                dx0[j] = dx
        else:
            gw = stage_W(kind, caches.pop((i, j)), gcaches.pop((i, j)))
            for l, g in enumerate(gw):
                for name, val in g.items():
                    grads[i][l][name] += val
    return loss, grads, dx0


def full_batch(kind, params, xs, tgts, H=None, dtype=np.float64):
    """Plain definition: all N microbatches as one batch, one unsplit forward and
    backward (monolithic: B immediately followed by W), gradient of
    L = (1/N) sum_j L_j."""
    params = _cast(params, dtype)
    N = len(xs)
    X = np.concatenate([np.asarray(x, dtype=dtype) for x in xs], axis=0)
    Tg = np.concatenate([np.asarray(t, dtype=dtype) for t in tgts], axis=0)
    stage_caches = []
    for sp in params:
        X, cch = stage_F(kind, sp, X, H)
        stage_caches.append(cch)
    n = X.size
    loss = 0.5 * ((X - Tg) ** 2).sum() / n
    dy = (X - Tg) / n
    grads = []
    for i in range(len(params) - 1, -1, -1):
        dy, gc = stage_B(kind, params[i], stage_caches[i], dy, H)
        grads.insert(0, stage_W(kind, stage_caches[i], gc))
    return loss, grads, dy


def global_order(X):
    """Flatten per-stage timed schedules (oracle.sched.Op lists) into one global
    execution order by start time (ties: stage index)."""
    ev = []
    for i, ops in enumerate(X):
        for op in ops:
            ev.append((op.start, i, op.kind, op.mb))
    ev.sort()
    return [(i, k, j) for (_s, i, k, j) in ev]


def merged_order(X):
    """Like global_order for a merge_w (1F1B) schedule: every B is followed by its W."""
    out = []
    for (i, k, j) in global_order(X):
        out.append((i, k, j))
        if k == "B":
            out.append((i, "W", j))
    return out
