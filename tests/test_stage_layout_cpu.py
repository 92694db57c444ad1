"""Stage shape validation (host code, no GPU): bf16 stages take the tcgen05
path whose fused attention is built for head dim 128 (GPT-2 shapes)
and T % 128 == 0; anything else is rejected up front (EINVAL / -1) instead of
running an untested path.  fp32 parity mode takes any head dim multiple of 8."""
import ctypes as C

import pytest

from paper_2504_19232_b200 import _lib as L


def _desc(dtype, d, H, T):
    s = L.StageDesc()
    s.block, s.dtype, s.n_layers, s.d, s.d_ff, s.n_heads = L.BLOCK_GPT, dtype, 1, d, 4 * d, H
    s.b, s.T, s.is_first, s.is_last, s.n_microbatches, s.n_slots, s.n_slots_fb = 1, T, 0, 0, 2, 2, 2
    return s


@pytest.mark.parametrize("dtype,d,H,T,ok", [
    (L.BF16, 256, 2, 128, True),      # dh 128
    (L.BF16, 2048, 16, 2048, True),   # C1
    (L.BF16, 256, 4, 128, False),     # dh 64
    (L.BF16, 512, 2, 128, False),     # dh 256
    (L.BF16, 256, 2, 200, False),     # T % 128
    (L.F32, 256, 4, 128, True),       # fp32: any dh % 8 == 0
    (L.F32, 128, 2, 64, True),
])
def test_bf16_requires_head_dim_128(dtype, d, H, T, ok):
    lib = L.lib()
    v = lib.adaptra_stage_slot_bytes(C.byref(_desc(dtype, d, H, T)))
    assert (v > 0) == ok
