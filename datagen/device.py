"""Device twin of the generator (datagen/gen.cu -> datagen/libdatagen.so).

Fills torch CUDA tensors with exactly the values ``datagen.tensor`` produces
on the host (bit-identical; see tests/test_gpu_parity.py).  No attention
arithmetic lives here."""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import INV_SIGMA_F32, stream_key

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdatagen.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise RuntimeError(f"{_LIB} missing: run python -m paper_2510_08726_b200.build")
        _lib = ctypes.CDLL(_LIB)
        _lib.datagen_fill.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_ulonglong, ctypes.c_longlong,
                                      ctypes.c_int, ctypes.c_float, ctypes.c_void_p]
        _lib.datagen_fill.restype = ctypes.c_int
    return _lib


def fill_(t: torch.Tensor, seed: int, tensor_id: int, start: int = 0) -> torch.Tensor:
    """Fill a contiguous CUDA tensor (bf16 or fp32) with elements [start, start + numel)."""
    if not (t.is_cuda and t.is_contiguous() and t.dtype in (torch.bfloat16, torch.float16, torch.float32)):
        raise ValueError("need a contiguous bf16/fp16/fp32 CUDA tensor")
    err = _load().datagen_fill(t.data_ptr(), t.numel(), stream_key(seed, tensor_id), start,
                               {torch.bfloat16: 1, torch.float16: 2}.get(t.dtype, 0), float(np.float32(INV_SIGMA_F32)),
                               ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    if err != 0:
        raise RuntimeError(f"datagen_fill failed with cudaError {err}")
    return t


def tensor(seed: int, tensor_id: int, shape, dtype=torch.bfloat16, device="cuda") -> torch.Tensor:
    return fill_(torch.empty(shape, dtype=dtype, device=device), seed, tensor_id)


def to_device(x: np.ndarray, device="cuda", dtype: str = "bf16") -> torch.Tensor:
    """Upload host generator output (uint16 bf16/fp16 bits or fp32) unchanged."""
    if x.dtype == np.uint16:
        tdt = torch.float16 if dtype == "f16" else torch.bfloat16
        return torch.from_numpy(x.view(np.int16).copy()).view(tdt).to(device)
    return torch.from_numpy(np.ascontiguousarray(x)).to(device)


def rising_logits_(q: torch.Tensor, k: torch.Tensor, amp: float, rate: float, tile: int = 128,
                   descending: bool = False):
    """In-place device twin of ``datagen.rising_logits`` (bit-identical values)."""
    from . import rising_rows
    sq, skv = q.shape[-2], k.shape[-2]
    rows = torch.from_numpy(rising_rows(sq)).to(q.device)
    qa = torch.where(rows, torch.tensor(amp, dtype=torch.float32, device=q.device),
                     torch.tensor(0.0, dtype=torch.float32, device=q.device))
    j = torch.arange(skv, dtype=torch.float64, device=k.device)
    if descending:
        j = (skv - 1) - j
    ka = (float(rate) * j / tile).to(torch.float32)
    q[..., 0] = qa.to(q.dtype)
    k[..., 0] = ka.to(k.dtype)
    return q, k
