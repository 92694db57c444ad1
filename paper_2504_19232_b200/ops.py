"""Thin torch-facing wrappers over the C-ABI (marshalling only)."""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return L.BF16
    if t.dtype == torch.float32:
        return L.F32
    raise TypeError(f"unsupported dtype {t.dtype}")


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def gemm(A, B, C_out, *, M, N, K, a_mn=0, b_mn=0, lda=None, ldb=None, ldc=None, Z=1, zdiv=1,
         a_off=(0, 0, 0, 0), b_off=(0, 0, 0, 0), c_off=(0, 0), epi=L.EPI_STORE, alpha=1.0,
         bias=None, aux=None, ldaux=None, aux_off=(0, 0), R=None, ldr=None, rowv=None, rowv_off=(0, 0),
         causal=L.CAUSAL_NONE, a_shape=None, b_shape=None, stream=None):
    """C[m,n] = sum_k A(m,k) B(n,k) (+ fused epilogue), see adaptra_gemm_desc_t.

    A, B are 2-D stored matrices; a_mn/b_mn select K-major (0) or MN-major (1)
    addressing; *_off = (row1, row2, col1, col2) batch offsets."""
    g = L.GemmDesc()
    g.dtype = _dt(A)
    g.M, g.N, g.K, g.Z, g.zdiv = M, N, K, Z, zdiv
    ar, ac = a_shape if a_shape else A.shape
    br, bc = b_shape if b_shape else B.shape
    g.A, g.lda, g.a_rows, g.a_cols = A.data_ptr(), lda or A.stride(0), ar, ac
    g.a_row1, g.a_row2, g.a_col1, g.a_col2 = a_off
    g.B, g.ldb, g.b_rows, g.b_cols = B.data_ptr(), ldb or B.stride(0), br, bc
    g.b_row1, g.b_row2, g.b_col1, g.b_col2 = b_off
    g.a_mn, g.b_mn = a_mn, b_mn
    g.epi, g.causal, g.alpha = epi, causal, alpha
    g.C, g.ldc = C_out.data_ptr(), ldc or C_out.stride(0)
    g.c_1, g.c_2 = c_off
    if aux is not None:
        g.aux, g.ldaux = aux.data_ptr(), ldaux or aux.stride(0)
        g.aux_1, g.aux_2 = aux_off
    if R is not None:
        g.R, g.ldr = R.data_ptr(), ldr or R.stride(0)
    if bias is not None:
        g.bias = bias.data_ptr()
    if rowv is not None:
        g.rowv = rowv.data_ptr()
        g.rowv_1, g.rowv_2 = rowv_off
    L.check(L.lib().adaptra_gemm(C.byref(g), _stream(stream)))
