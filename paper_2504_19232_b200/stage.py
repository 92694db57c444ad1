"""torch-owned buffers + C-ABI handle for one pipeline stage (marshalling only).

Buffer layouts are those of include/adaptra.h (adaptra_stage_desc_t).  Packing
parameters from per-layer dicts into the flat buffers happens once at setup.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L

GPT_W = ("Wqkv", "Wo", "W1", "W2")
GPT_V = ("ln1_g", "ln1_b", "bqkv", "bo", "ln2_g", "ln2_b", "b1", "b2")
MLP_W = ("W1", "W2")
MLP_V = ("b1", "b2")

TORCH_DT = {L.F32: torch.float32, L.BF16: torch.bfloat16}


class Stage:
    def __init__(self, block, dtype, n_layers, d, d_ff, n_heads, b, T, is_first, is_last, n_microbatches,
                 n_slots, device, n_slots_fb=None):
        self.block, self.dtype = block, dtype
        self.n_layers, self.d, self.d_ff, self.n_heads, self.b, self.T = n_layers, d, d_ff, n_heads, b, T
        self.is_first, self.is_last = is_first, is_last
        self.device = torch.device(device)
        self.tdt = TORCH_DT[dtype]
        desc = L.StageDesc()
        desc.block, desc.dtype = block, dtype
        desc.n_layers, desc.d, desc.d_ff, desc.n_heads = n_layers, d, d_ff, n_heads
        desc.b, desc.T, desc.is_first, desc.is_last = b, T, int(is_first), int(is_last)
        desc.n_microbatches, desc.n_slots = n_microbatches, n_slots
        desc.n_slots_fb = n_slots_fb or n_slots
        lib = L.lib()
        nw = lib.adaptra_stage_wts_elems(C.byref(desc))
        nv = lib.adaptra_stage_vecs_elems(C.byref(desc))
        sb = lib.adaptra_stage_slot_bytes(C.byref(desc))
        wb = lib.adaptra_stage_work_bytes(C.byref(desc))
        fb = lib.adaptra_stage_slot_fb_bytes(C.byref(desc))
        if sb < 0 or wb < 0 or fb < 0:
            L.check(L.EINVAL)
        self.slot_bytes, self.work_bytes, self.slot_fb_bytes = sb, wb, fb
        self.n_slots, self.n_slots_fb = n_slots, desc.n_slots_fb
        dev = self.device
        self.wts = torch.zeros(nw, dtype=self.tdt, device=dev)
        self.vecs = torch.zeros(nv, dtype=torch.float32, device=dev)
        self.gwts = torch.zeros(nw, dtype=torch.float32, device=dev)
        self.gvecs = torch.zeros(nv, dtype=torch.float32, device=dev)
        self.stash = torch.empty(n_slots * sb, dtype=torch.uint8, device=dev)
        self.stash_fb = torch.empty(desc.n_slots_fb * fb, dtype=torch.uint8, device=dev)
        self.work = torch.empty(max(wb, 256), dtype=torch.uint8, device=dev)
        desc.wts, desc.vecs = self.wts.data_ptr(), self.vecs.data_ptr()
        desc.gwts, desc.gvecs = self.gwts.data_ptr(), self.gvecs.data_ptr()
        desc.stash, desc.work = self.stash.data_ptr(), self.work.data_ptr()
        desc.stash_fb = self.stash_fb.data_ptr()
        self.desc = desc
        h = C.c_void_p()
        L.check(lib.adaptra_stage_create(C.byref(desc), C.byref(h)))
        self.handle = h

    # ------------------------------------------------------------ params
    def _names(self):
        return (GPT_W, GPT_V) if self.block == L.BLOCK_GPT else (MLP_W, MLP_V)

    def load_params(self, layers):
        """layers: list of dicts of numpy arrays (weights [out, in])."""
        wn, vn = self._names()
        w = np.concatenate([np.asarray(p[k], np.float32).ravel() for p in layers for k in wn])
        v = np.concatenate([np.asarray(p[k], np.float32).ravel() for p in layers for k in vn])
        self.wts.copy_(torch.from_numpy(w).to(self.tdt))
        self.vecs.copy_(torch.from_numpy(v))

    def _unpack(self, flat_w, flat_v):
        wn, vn = self._names()
        d, f = self.d, self.d_ff
        wshape = {"Wqkv": (3 * d, d), "Wo": (d, d), "W1": (f, d), "W2": (d, f)}
        vshape = {"ln1_g": d, "ln1_b": d, "bqkv": 3 * d, "bo": d, "ln2_g": d, "ln2_b": d, "b1": f, "b2": d}
        out = []
        ow = ov = 0
        for _ in range(self.n_layers):
            p = {}
            for k in wn:
                n = wshape[k][0] * wshape[k][1]
                p[k] = flat_w[ow:ow + n].reshape(wshape[k])
                ow += n
            for k in vn:
                n = vshape[k]
                p[k] = flat_v[ov:ov + n]
                ov += n
            out.append(p)
        return out

    def grads(self):
        return self._unpack(self.gwts.double().cpu().numpy(), self.gvecs.double().cpu().numpy())

    # ------------------------------------------------------------ ops
    @staticmethod
    def _s(stream):
        s = stream if stream is not None else torch.cuda.current_stream()
        return C.c_void_p(s.cuda_stream)

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr() if t is not None else 0)

    def F(self, slot, x_in, y_out=None, target=None, loss_acc=None, stream=None):
        L.check(L.lib().adaptra_stage_F(self.handle, slot, self._p(x_in), self._p(y_out), self._p(target),
                                        self._p(loss_acc), self._s(stream)))

    def B(self, slot, dy_in=None, dx_out=None, stream=None):
        L.check(L.lib().adaptra_stage_B(self.handle, slot, self._p(dy_in), self._p(dx_out), self._s(stream)))

    def W(self, slot, stream=None):
        L.check(L.lib().adaptra_stage_W(self.handle, slot, self._s(stream)))

    def W2(self, slot_a, slot_b, stream=None):
        """W of two slots as one launch (K = 2bT), adaptra_stage_W2."""
        L.check(L.lib().adaptra_stage_W2(self.handle, slot_a, slot_b, self._s(stream)))

    def Wn(self, slots, stream=None):
        """W of 1..4 slots as one launch (K = n bT), adaptra_stage_Wn."""
        arr = (C.c_int32 * len(slots))(*slots)
        L.check(L.lib().adaptra_stage_Wn(self.handle, arr, len(slots), self._s(stream)))

    def zero_grads(self, stream=None):
        L.check(L.lib().adaptra_stage_zero_grads(self.handle, self._s(stream)))

    def act(self):
        """A new activation buffer [b*T, d] in the stage dtype."""
        return torch.empty(self.b * self.T, self.d, dtype=self.tdt, device=self.device)

    def close(self):
        if self.handle:
            L.lib().adaptra_stage_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
