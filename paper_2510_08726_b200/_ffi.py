"""ctypes mirror of include/attn.h.  Loading fails loudly: there is no
fallback implementation anywhere in this package."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# ATTN_LIB_PATH overrides the in-tree library (developer A/B builds only).
LIB_PATH = os.environ.get("ATTN_LIB_PATH") or os.path.join(_HERE, "libattn.so")

ATTN_OK = 0
ATTN_ERR_INVALID_ARGUMENT = 1
ATTN_ERR_UNSUPPORTED = 2
ATTN_ERR_ALIGNMENT = 3
ATTN_ERR_WORKSPACE_TOO_SMALL = 4
ATTN_ERR_CUDA = 5
ATTN_ERR_NCCL = 6
ATTN_BF16 = 0
ATTN_FP32 = 1
ATTN_FP16 = 2
ATTN_Q_POS_DEFAULT = -(1 << 63)

EXPORTED = ("attn_fused_fwd", "attn_splitkv_default_splits", "attn_splitkv_workspace_bytes",
            "attn_splitkv_decode", "attn_combine", "attn_status_string", "attn_last_error",
            "attn_abi_version", "attn_last_launch_count", "attn_merge_partials", "attn_softmax_rows",
            "attn_nccl_get_unique_id", "attn_nccl_comm_init", "attn_nccl_comm_destroy",
            "attn_decode_kv_sharded_workspace_bytes", "attn_decode_kv_sharded",
            "attn_fused_fwd_default_splits", "attn_fused_fwd_workspace_bytes", "attn_fused_fwd_splitkv",
            "attn_debug_repair_counters", "attn_fused_fwd_partial", "attn_splitkv_decode_packed")
# repair-event counter slots (include/attn.h ATTN_REPAIR_*)
ATTN_REPAIR_FWD128, ATTN_REPAIR_FWD64, ATTN_REPAIR_PERSIST, ATTN_REPAIR_DECODE = 0, 1, 2, 3
ATTN_REPAIR_SLOTS = 4


class AttnTensor(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("stride_b", ctypes.c_int64), ("stride_h", ctypes.c_int64),
                ("stride_s", ctypes.c_int64)]


class AttnProblem(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("heads_q", ctypes.c_int32), ("heads_kv", ctypes.c_int32),
                ("seqlen_q", ctypes.c_int32), ("seqlen_kv", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("scale", ctypes.c_float), ("softcap", ctypes.c_float),
                ("alibi_slopes", ctypes.c_void_p), ("causal", ctypes.c_int32), ("window_left", ctypes.c_int32),
                ("window_right", ctypes.c_int32), ("seqlen_kv_total", ctypes.c_int64),
                ("q_pos_offset", ctypes.c_int64), ("kv_pos_offset", ctypes.c_int64)]


class AttnParts(ctypes.Structure):
    _fields_ = [("m", ctypes.c_void_p), ("l", ctypes.c_void_p), ("o", ctypes.c_void_p),
                ("num_parts", ctypes.c_int32), ("m_stride_part", ctypes.c_int64), ("m_stride_b", ctypes.c_int64),
                ("m_stride_h", ctypes.c_int64), ("o_stride_part", ctypes.c_int64), ("o_stride_b", ctypes.c_int64),
                ("o_stride_h", ctypes.c_int64)]


_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libattn.so (built in-tree by ``paper_2510_08726_b200/build.py``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: run `python -m paper_2510_08726_b200.build` "
                           "(there is no fallback implementation)")
    lib = ctypes.CDLL(path)
    if os.environ.get("ATTN_LIB_PATH"):
        # developer A/B builds of older revisions may lack newer entry points: bind what exists
        class _Partial:
            def __init__(self, l):
                self.__dict__["_l"] = l

            def __getattr__(self, n):
                try:
                    return getattr(self._l, n)
                except AttributeError:
                    return ctypes.CFUNCTYPE(ctypes.c_int)(lambda *a: 2)

            def __setattr__(self, n, v):
                pass
        missing = [n for n in EXPORTED if not hasattr(lib, n)]
        if missing:
            lib = _Partial(lib)
    P, T, Pa = ctypes.POINTER(AttnProblem), AttnTensor, ctypes.POINTER(AttnParts)
    vp, i32, f32p = ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p
    lib.attn_fused_fwd.argtypes = [P, T, T, T, T, f32p, vp]
    lib.attn_fused_fwd.restype = ctypes.c_int
    lib.attn_fused_fwd_default_splits.argtypes = [P, i32]
    lib.attn_fused_fwd_default_splits.restype = i32
    lib.attn_fused_fwd_workspace_bytes.argtypes = [P, i32]
    lib.attn_fused_fwd_workspace_bytes.restype = ctypes.c_size_t
    lib.attn_fused_fwd_splitkv.argtypes = [P, T, T, T, T, f32p, i32, vp, ctypes.c_size_t, vp]
    lib.attn_fused_fwd_splitkv.restype = ctypes.c_int
    lib.attn_fused_fwd_partial.argtypes = [P, T, T, T, vp, vp, vp]
    lib.attn_fused_fwd_partial.restype = ctypes.c_int
    lib.attn_splitkv_default_splits.argtypes = [P, i32]
    lib.attn_splitkv_default_splits.restype = i32
    lib.attn_splitkv_workspace_bytes.argtypes = [P, i32]
    lib.attn_splitkv_workspace_bytes.restype = ctypes.c_size_t
    lib.attn_splitkv_decode.argtypes = [P, T, T, T, i32, vp, ctypes.c_size_t, Pa, T, f32p, vp]
    lib.attn_splitkv_decode.restype = ctypes.c_int
    lib.attn_splitkv_decode_packed.argtypes = [P, T, T, T, i32, vp, ctypes.c_size_t, vp, vp]
    lib.attn_splitkv_decode_packed.restype = ctypes.c_int
    lib.attn_combine.argtypes = [i32, i32, i32, Pa, ctypes.c_int, T, f32p, Pa, vp]
    lib.attn_combine.restype = ctypes.c_int
    i64 = ctypes.c_int64
    lib.attn_merge_partials.argtypes = [i32, i64, i32, ctypes.c_int, vp, i64, i64, vp, i64, ctypes.c_int, vp, i64, vp,
                                        vp]
    lib.attn_merge_partials.restype = ctypes.c_int
    lib.attn_softmax_rows.argtypes = [i64, i32, ctypes.c_int, vp, i64, vp, i64, vp, vp, vp]
    lib.attn_softmax_rows.restype = ctypes.c_int
    lib.attn_nccl_get_unique_id.argtypes = [vp]
    lib.attn_nccl_get_unique_id.restype = ctypes.c_int
    lib.attn_nccl_comm_init.argtypes = [ctypes.POINTER(ctypes.c_void_p), i32, i32, vp]
    lib.attn_nccl_comm_init.restype = ctypes.c_int
    lib.attn_nccl_comm_destroy.argtypes = [vp]
    lib.attn_nccl_comm_destroy.restype = ctypes.c_int
    lib.attn_decode_kv_sharded_workspace_bytes.argtypes = [P, i32]
    lib.attn_decode_kv_sharded_workspace_bytes.restype = ctypes.c_size_t
    lib.attn_decode_kv_sharded.argtypes = [vp, P, T, T, T, vp, ctypes.c_size_t, T, f32p, vp]
    lib.attn_decode_kv_sharded.restype = ctypes.c_int
    lib.attn_status_string.argtypes = [ctypes.c_int]
    lib.attn_status_string.restype = ctypes.c_char_p
    lib.attn_last_error.restype = ctypes.c_char_p
    lib.attn_abi_version.restype = ctypes.c_int
    lib.attn_last_launch_count.restype = ctypes.c_int
    lib.attn_debug_repair_counters.argtypes = [vp]
    lib.attn_debug_repair_counters.restype = None
    if lib.attn_abi_version() != 1:
        raise RuntimeError("libattn.so ABI version mismatch")
    _lib = lib
    return lib


class AttnError(RuntimeError):
    def __init__(self, status: int, what: str):
        lib = load()
        super().__init__(f"{what}: {lib.attn_status_string(status).decode()} "
                         f"({lib.attn_last_error().decode()})")
        self.status = status


def check(status: int, what: str) -> None:
    if status != ATTN_OK:
        raise AttnError(status, what)
