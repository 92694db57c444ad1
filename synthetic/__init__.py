"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic: it only draws random numbers
(numpy PCG64, fixed seeds) with the shapes and distributions of the paper's
GPT-2 workloads (DESIGN.md §4 "input recipe"), and the straggler trace of the
paper's appendix table.  Both ``oracle/`` and the product path's
tests/bench take their inputs from here; neither imports the other.
"""
from __future__ import annotations

import numpy as np

MLP_NAMES = ("W1", "b1", "W2", "b2")
GPT_NAMES = ("ln1_g", "ln1_b", "Wqkv", "bqkv", "Wo", "bo",
             "ln2_g", "ln2_b", "W1", "b1", "W2", "b2")


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16-representable float32 (RNE), so
    that a bf16 run and a float64 oracle start from identical values."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return rounded.astype(np.uint32).view(np.float32).reshape(a.shape)


def mlp_params(seed: int, S: int, L: int, d: int, dff: int, bf16: bool = False):
    """params[stage][layer] dict for the C0 MLP block (weights [out, in])."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(S):
        st = []
        for _ in range(L):
            p = {
                "W1": rng.normal(0.0, 1.0 / np.sqrt(d), (dff, d)).astype(np.float32),
                "b1": rng.normal(0.0, 0.1, (dff,)).astype(np.float32),
                "W2": rng.normal(0.0, 1.0 / np.sqrt(dff), (d, dff)).astype(np.float32),
                "b2": rng.normal(0.0, 0.1, (d,)).astype(np.float32),
            }
            if bf16:
                p = {k: round_bf16(v) for k, v in p.items()}
            st.append(p)
        out.append(st)
    return out


def gpt_params(seed: int, S: int, L: int, d: int, dff: int, perturb: bool = True,
               bf16: bool = False, n_layers_total: int | None = None):
    """params[stage][layer] for the GPT-2 pre-LN block.

    GPT-2 init: weights N(0, 0.02), output projections (Wo, W2) scaled by
    1/sqrt(2 n_layers); LN gamma = 1, beta = 0; biases 0.  ``perturb`` adds
    small random biases / LN affine terms so that every parameter matters in
    parity tests.
    """
    rng = np.random.default_rng(seed)
    nl = n_layers_total or S * L
    ro = 0.02 / np.sqrt(2 * nl)
    out = []
    for _ in range(S):
        st = []
        for _ in range(L):
            p = {
                "ln1_g": np.ones(d, np.float32), "ln1_b": np.zeros(d, np.float32),
                "Wqkv": rng.normal(0.0, 0.02, (3 * d, d)).astype(np.float32),
                "bqkv": np.zeros(3 * d, np.float32),
                "Wo": rng.normal(0.0, ro, (d, d)).astype(np.float32),
                "bo": np.zeros(d, np.float32),
                "ln2_g": np.ones(d, np.float32), "ln2_b": np.zeros(d, np.float32),
                "W1": rng.normal(0.0, 0.02, (dff, d)).astype(np.float32),
                "b1": np.zeros(dff, np.float32),
                "W2": rng.normal(0.0, ro, (d, dff)).astype(np.float32),
                "b2": np.zeros(d, np.float32),
            }
            if perturb:
                for k in ("ln1_g", "ln2_g"):
                    p[k] = (1.0 + rng.normal(0.0, 0.1, d)).astype(np.float32)
                for k in ("ln1_b", "ln2_b", "bqkv", "bo", "b1", "b2"):
                    p[k] = rng.normal(0.0, 0.05, p[k].shape).astype(np.float32)
                # larger projections so attention is not uniform at small d
                p["Wqkv"] = rng.normal(0.0, 1.0 / np.sqrt(d), (3 * d, d)).astype(np.float32)
                p["Wo"] = rng.normal(0.0, 0.5 / np.sqrt(d), (d, d)).astype(np.float32)
                p["W1"] = rng.normal(0.0, 1.0 / np.sqrt(d), (dff, d)).astype(np.float32)
                p["W2"] = rng.normal(0.0, 0.5 / np.sqrt(dff), (d, dff)).astype(np.float32)
            if bf16:
                p = {k: (round_bf16(v) if v.ndim == 2 else v) for k, v in p.items()}
            st.append(p)
        out.append(st)
    return out


def microbatches(seed: int, N: int, b: int, T: int, d: int, bf16: bool = False):
    """N microbatches x_j ~ N(0, 1) of shape [b, T, d] (seed 1 in the bench)."""
    rng = np.random.default_rng(seed)
    xs = [rng.normal(0.0, 1.0, (b, T, d)).astype(np.float32) for _ in range(N)]
    if bf16:
        xs = [round_bf16(x) for x in xs]
    return xs


def targets(seed: int, N: int, b: int, T: int, d: int):
    """MSE targets ~ N(0, 1) (seed 2 in the bench); float32 on both sides."""
    rng = np.random.default_rng(seed)
    return [rng.normal(0.0, 1.0, (b, T, d)).astype(np.float32) for _ in range(N)]


def stage_profile(seed: int, S: int, lo: int = 5, hi: int = 20, c_hi: int = 0):
    """Random integer per-stage op times and link latencies for schedule tests."""
    rng = np.random.default_rng(seed)
    tF = [int(v) for v in rng.integers(lo, hi + 1, S)]
    tB = [int(v) for v in rng.integers(lo, hi + 1, S)]
    tW = [int(v) for v in rng.integers(lo, hi + 1, S)]
    c = [int(v) for v in rng.integers(0, c_hi + 1, S - 1)] if c_hi > 0 else [0] * (S - 1)
    return tF, tB, tW, c


# Appendix table "Injected trace of communication stragglers".
# Ranges are half-open iterations [from, to) (R17); "a<->a+1" is link a;
# event 9 is an RNIC failure on link 2 from iteration 1030 to the end (1200).
PAPER_TRACE = [
    {"id": 0, "from": 15, "to": 85, "links": [2], "latency_ms": 30},
    {"id": 1, "from": 120, "to": 190, "links": [0, 5], "latency_ms": 40},
    {"id": 2, "from": 230, "to": 300, "links": [6], "latency_ms": 20},
    {"id": 3, "from": 340, "to": 410, "links": [2, 3, 6], "latency_ms": 50},
    {"id": 4, "from": 450, "to": 520, "links": [5], "latency_ms": 60},
    {"id": 5, "from": 560, "to": 630, "links": [1, 6], "latency_ms": 60},
    {"id": 6, "from": 670, "to": 740, "links": [0, 4], "latency_ms": 20},
    {"id": 7, "from": 780, "to": 850, "links": [0, 1, 2], "latency_ms": 40},
    {"id": 8, "from": 890, "to": 960, "links": [4, 5], "latency_ms": 50},
    {"id": 9, "from": 1030, "to": 1200, "links": [2], "latency_ms": float("inf")},
]
PAPER_TRACE_ITERS = 1200
