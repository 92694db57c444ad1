"""ctypes binding of libadaptra.so (include/adaptra.h).  Argument marshalling
only: every step of the path runs in the library's kernels / host code.

The product path fails loudly when the library is missing: there is no CPU or
PyTorch fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libadaptra.so")

OK = 0
EINVAL, EPLAN, EDEADLOCK, ECUDA, ENOMEM, ELINK, ETOOBIG = -1, -2, -3, -4, -5, -6, -7

OP_F, OP_B, OP_W = 0, 1, 2
SEL_PAPER, SEL_CAP, MERGE_W = 0, 1, 2
TUNE_GEMM_SMS = 1
TUNE_ATTN_SMS = 2
EXEC_INORDER = 16
EXEC_NCCL = 32
NCCL_ID_BYTES = 128
F32, BF16 = 0, 1
BLOCK_MLP, BLOCK_GPT = 0, 1

EPI_STORE, EPI_GELU, EPI_RESID, EPI_DGELU, EPI_ACC_F32, EPI_STORE_F32, EPI_DSOFTMAX = range(7)
CAUSAL_NONE, CAUSAL_TILE, CAUSAL_KEND, CAUSAL_KSTART = range(4)

LINK_DIRECT, LINK_P2P, LINK_HOST = 0, 1, 2
PATH_GPU, PATH_HOST = 0, 1
IPC_BYTES = 128
LINK_DOWN = (1 << 63) - 1

_i32, _i64, _u32, _f32, _vp = C.c_int32, C.c_int64, C.c_uint32, C.c_float, C.c_void_p


class AdaptraError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"adaptra error {code}: {msg}")
        self.code = code


class Op(C.Structure):
    _fields_ = [("kind", _i32), ("mb", _i32), ("start", _i64), ("end", _i64)]


class Violation(C.Structure):
    _fields_ = [("code", _i32), ("stage", _i32), ("kind", _i32), ("mb", _i32)]


V_CODES = {1: "badop", 2: "dup", 3: "missing", 4: "duration", 5: "overlap", 6: "dep",
           7: "nonmono", 8: "x_last", 9: "x0_gt_N"}
ARM_1F1B, ARM_ZB, ARM_ADAPTIVE = 0, 1, 2
MAX_STAGES = 64


class PlannerDesc(C.Structure):
    _fields_ = [("S", _i32), ("N", _i32), ("arm", _i32), ("ratio", _i32),
                ("tF", C.POINTER(_i64)), ("tB", C.POINTER(_i64)), ("tW", C.POINTER(_i64)),
                ("x_init", C.POINTER(_i32)), ("x_cap", C.POINTER(_i32)),
                ("mem_capacity", _i64), ("mem_per_act", _i64)]


class PlanInfo(C.Structure):
    _fields_ = [("makespan", _i64), ("delta", _i64), ("replans", _i64),
                ("tF", _i64 * MAX_STAGES), ("tB", _i64 * MAX_STAGES), ("tW", _i64 * MAX_STAGES)]


class GemmDesc(C.Structure):
    _fields_ = [
        ("dtype", _i32), ("M", _i32), ("N", _i32), ("K", _i32), ("Z", _i32), ("zdiv", _i32),
        ("A", _vp), ("lda", _i64), ("a_rows", _i64), ("a_cols", _i64),
        ("a_row1", _i64), ("a_row2", _i64), ("a_col1", _i64), ("a_col2", _i64),
        ("a_mn", _i32), ("b_mn", _i32),
        ("B", _vp), ("ldb", _i64), ("b_rows", _i64), ("b_cols", _i64),
        ("b_row1", _i64), ("b_row2", _i64), ("b_col1", _i64), ("b_col2", _i64),
        ("epi", _i32), ("causal", _i32), ("alpha", _f32), ("pad0", _i32),
        ("C", _vp), ("ldc", _i64), ("c_1", _i64), ("c_2", _i64),
        ("aux", _vp), ("ldaux", _i64), ("aux_1", _i64), ("aux_2", _i64),
        ("R", _vp), ("ldr", _i64), ("bias", _vp), ("rowv", _vp), ("rowv_1", _i64), ("rowv_2", _i64),
    ]


class StageDesc(C.Structure):
    _fields_ = [
        ("block", _i32), ("dtype", _i32), ("n_layers", _i32), ("d", _i32), ("d_ff", _i32), ("n_heads", _i32),
        ("b", _i32), ("T", _i32), ("is_first", _i32), ("is_last", _i32), ("n_microbatches", _i32),
        ("n_slots", _i32), ("n_slots_fb", _i32), ("wts", _vp), ("vecs", _vp), ("gwts", _vp), ("gvecs", _vp),
        ("stash", _vp), ("stash_fb", _vp), ("work", _vp),
    ]


class ExecDesc(C.Structure):
    _fields_ = [
        ("stage", _vp), ("stage_index", _i32), ("n_stages", _i32), ("n_microbatches", _i32),
        ("in_fwd", _vp), ("in_bwd", _vp), ("out_fwd", _vp), ("out_bwd", _vp), ("compute_stream", _vp),
        ("inputs", C.POINTER(_vp)), ("targets", C.POINTER(_vp)), ("loss_acc", _vp),
    ]


class IterStats(C.Structure):
    _fields_ = [("n_ops", _i64), ("busy_ns", _i64), ("first_start_ns", _i64), ("last_end_ns", _i64),
                ("op_ns", _i64 * 3), ("op_cnt", _i64 * 3), ("host_enqueue_ns", _i64)]


_P = C.POINTER
_SIGS = {
    "adaptra_last_error": (C.c_char_p, []),
    "adaptra_version": (C.c_char_p, []),
    "adaptra_plan_init": (_i32, [_i32, _i32, _i64, _i64, _P(_i32)]),
    "adaptra_plan_adapt": (_i32, [_i32, _i32, _P(_i64), _P(_i64), _P(_i64), _P(_i32)]),
    "adaptra_eq1_holds": (_i32, [_i32, _P(_i64), _P(_i64), _P(_i64), _P(_i32), _P(C.c_uint8)]),
    "adaptra_schedule": (_i32, [_i32, _i32, _P(_i64), _P(_i64), _P(_i64), _P(_i64), _P(_i32), _i64, _u32,
                                _P(Op), _P(_i32), _P(_i64), _P(_i64)]),
    "adaptra_replay": (_i32, [_i32, _i32, _P(_i64), _P(_i64), _P(_i64), _P(_i64), _P(Op), _P(_i32), _u32,
                              _P(Op), _P(_i64)]),
    "adaptra_validate": (_i32, [_i32, _i32, _P(_i64), _P(_i64), _P(_i64), _P(_i64), _P(Op), _P(_i32), _u32,
                                _P(Violation), _i32, _P(_i32)]),
    "adaptra_validate_plan": (_i32, [_i32, _i32, _P(_i32), _P(Violation), _i32, _P(_i32)]),
    "adaptra_plan_1f1b": (_i32, [_i32, _i32, _P(_i32)]),
    "adaptra_clamp_plan": (_i32, [_i32, _P(_i32), _P(_i32)]),
    "adaptra_default_delta": (_i64, [_i32, _P(_i64), _P(_i64), _P(_i64), _i32]),
    "adaptra_planner_create": (_i32, [_P(PlannerDesc), _P(_vp)]),
    "adaptra_planner_destroy": (_i32, [_vp]),
    "adaptra_planner_set_profile": (_i32, [_vp, _P(_i64), _P(_i64), _P(_i64)]),
    "adaptra_planner_step": (_i32, [_vp, _P(_i64), _P(Op), _P(_i32), _P(_i32), _P(_i32), _P(PlanInfo)]),
    "adaptra_gemm": (_i32, [_P(GemmDesc), _vp]),
    "adaptra_set_tuning": (_i32, [_i32, _i64]),
    "adaptra_prof_enable": (_i32, [_i32]),
    "adaptra_launch_count": (_i64, []),
    "adaptra_p2p_copy": (_i32, [C.c_void_p, C.c_void_p, _i64, C.c_void_p]),
    "adaptra_prof_collect": (_i32, [_i32, _P(_i64), _P(C.c_double), _P(C.c_double), _P(C.c_double)]),
    "adaptra_prof_collect_ex": (_i32, [_i32, _P(_i64), _P(C.c_double), _P(C.c_double), _P(C.c_double),
                                       _P(C.c_double)]),
    "adaptra_stage_slot_bytes": (_i64, [_P(StageDesc)]),
    "adaptra_stage_slot_fb_bytes": (_i64, [_P(StageDesc)]),
    "adaptra_stage_work_bytes": (_i64, [_P(StageDesc)]),
    "adaptra_stage_wts_elems": (_i64, [_P(StageDesc)]),
    "adaptra_stage_vecs_elems": (_i64, [_P(StageDesc)]),
    "adaptra_stage_create": (_i32, [_P(StageDesc), _P(_vp)]),
    "adaptra_stage_destroy": (_i32, [_vp]),
    "adaptra_stage_F": (_i32, [_vp, _i32, _vp, _vp, _vp, _vp, _vp]),
    "adaptra_stage_B": (_i32, [_vp, _i32, _vp, _vp, _vp]),
    "adaptra_stage_W": (_i32, [_vp, _i32, _vp]),
    "adaptra_stage_W2": (_i32, [_vp, _i32, _i32, _vp]),
    "adaptra_stage_Wn": (_i32, [_vp, _P(_i32), _i32, _vp]),
    "adaptra_stage_zero_grads": (_i32, [_vp, _vp]),
    "adaptra_inbox_create": (_i32, [_i32, _i32, _i64, C.c_char_p, _P(_vp)]),
    "adaptra_inbox_destroy": (_i32, [_vp]),
    "adaptra_inbox_export": (_i32, [_vp, _P(C.c_uint8)]),
    "adaptra_inbox_slot": (_vp, [_vp, _i32]),
    "adaptra_recv": (_i32, [_vp, _i32, _u32, _vp, _P(_vp)]),
    "adaptra_inbox_set_host": (_i32, [_vp, _i32]),
    "adaptra_inbox_poison": (_i32, [_vp]),
    "adaptra_inbox_reset": (_i32, [_vp]),
    "adaptra_outbox_open_local": (_i32, [_i32, _vp, _i32, _P(_vp)]),
    "adaptra_outbox_open_ipc": (_i32, [_i32, _P(C.c_uint8), _i32, _i64, C.c_char_p, _i32, _P(_vp)]),
    "adaptra_outbox_close": (_i32, [_vp]),
    "adaptra_outbox_dst": (_vp, [_vp, _i32]),
    "adaptra_set_link_latency": (_i32, [_vp, _i64]),
    "adaptra_link_set_path": (_i32, [_vp, _i32]),
    "adaptra_send": (_i32, [_vp, _i32, _vp, _u32]),
    "adaptra_recv_blocking": (_i32, [_vp, _i32, _u32, _P(_vp)]),
    "adaptra_send_wait": (_i32, [_vp, _i32, _u32]),
    "adaptra_link_stats": (_i32, [_vp, _P(_i64), _P(_i64), _P(_i64)]),
    "adaptra_link_stats_take": (_i32, [_vp, _P(_i64), _P(_i64), _P(_i64)]),
    "adaptra_exec_create": (_i32, [_P(ExecDesc), _P(_vp)]),
    "adaptra_exec_destroy": (_i32, [_vp]),
    "adaptra_run_iteration": (_i32, [_vp, _P(Op), _i32, _u32, _u32]),
    "adaptra_exec_set_time_base": (_i32, [_vp, _vp]),
    "adaptra_exec_set_host_io": (_i32, [_vp, _P(_vp), _i64, _vp]),
    "adaptra_exec_set_nccl": (_i32, [_vp, _vp, _i32, _i32, _i64]),
    "adaptra_nccl_post_plan": (_i32, [_i32, _P(Op), _P(_i32), _u32, _i32, _P(_i32)]),
    "adaptra_exec_set_nccl_post": (_i32, [_vp, _P(_i32), _i32]),
    "adaptra_nccl_p2p": (_i32, [_vp, _i32, _vp, _i64, _i32, _vp]),
    "adaptra_exec_set_offload": (_i32, [_vp, _vp, _i32, _i32]),
    "adaptra_exec_offload_stats": (_i32, [_vp, _P(_i32), _P(_i32), _P(_i64)]),
    "adaptra_offload_plan": (_i32, [_P(Op), _i32, _i32, _i32, _i32, _i32, _u32, _P(_i32), _P(_i32), _i32, _P(_i32)]),
    "adaptra_nccl_unique_id": (_i32, [_P(C.c_uint8)]),
    "adaptra_nccl_comm_init": (_i32, [_P(C.c_uint8), _i32, _i32, _i32, _P(_vp)]),
    "adaptra_nccl_comm_destroy": (_i32, [_vp]),
    "adaptra_exec_join": (_i32, [_vp]),
    "adaptra_exec_wait": (_i32, [_vp, _P(IterStats), _P(_i64)]),
    "adaptra_exec_profile": (_i32, [_vp, _i32, _i64, _P(_i64)]),
    "adaptra_median_ticks": (_i64, [_P(_i64), _i32, _i64]),
}

_lib = None


def declared_symbols():
    """Every entry point include/adaptra.h declares (the binding binds all)."""
    return list(_SIGS)


def lib():
    """Load libadaptra.so (in-tree).  Raises if it is missing: no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc):
    if rc != OK:
        msg = lib().adaptra_last_error()
        raise AdaptraError(rc, msg.decode() if msg else "")
    return rc
