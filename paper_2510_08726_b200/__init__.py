"""B200-native (sm_100a) hot path of Neptune (arXiv 2510.08726): fused
attention by Rolling Update (prefill) and Split-K Update (decode).

This module is argument marshalling only: every arithmetic step runs in the
CUDA kernels of ``libattn.so`` behind the C ABI in ``include/attn.h``.
PyTorch supplies device memory and streams.  There is no CPU fallback: if the
library is missing or a configuration is unsupported, the call raises.

Tensors use the BHSD layout of the paper's Fig. 8:
q [B, Hq, Sq, D], k/v [B, Hkv, Skv, D], D contiguous.
"""
from __future__ import annotations

import ctypes
import math
from typing import Optional, Tuple

import torch

from . import _ffi
from ._ffi import AttnParts, AttnProblem, AttnTensor, check, load

__all__ = ["fused_fwd", "fused_fwd_partial", "splitkv_decode", "combine", "merge_partials", "softmax_rows", "default_splits", "workspace_bytes",
           "last_launch_count", "Parts", "load", "repair_counters"]

_DT = {torch.bfloat16: _ffi.ATTN_BF16, torch.float32: _ffi.ATTN_FP32, torch.float16: _ffi.ATTN_FP16}


def _as_tensor(t: Optional[torch.Tensor]) -> AttnTensor:
    if t is None:
        return AttnTensor(None, 0, 0, 0)
    st = t.stride()
    if len(st) != 4 or st[3] != 1:
        raise ValueError("expected a [B, H, S, D] tensor with a contiguous last dimension")
    return AttnTensor(t.data_ptr(), st[0], st[1], st[2])


def _stream(stream) -> ctypes.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _check_io(q, k, v, out=None, lse=None, lse_shape=None):
    """Shape / dtype / device checks the C ABI cannot make (it sees only pointers and
    strides, not allocation sizes): a mismatch here would be an out-of-bounds device
    access, so it raises ValueError before anything is launched.  (Kept cheap: it runs on
    every call, and small calls are launch-bound.)"""
    qs, ks, vs = q.shape, k.shape, v.shape
    if len(qs) != 4 or len(ks) != 4:
        raise ValueError(f"q, k must be [B, H, S, D] tensors (got {tuple(qs)}, {tuple(ks)})")
    if vs != ks:
        raise ValueError(f"v {tuple(vs)} must have k's shape {tuple(ks)}")
    if ks[0] != qs[0] or ks[3] != qs[3]:
        raise ValueError("q and k disagree on batch or head_dim")
    if ks[1] < 1 or qs[1] % ks[1] != 0:
        raise ValueError(f"heads_q ({qs[1]}) must be a multiple of heads_kv ({ks[1]})")
    dt, dev = q.dtype, q.get_device()
    if k.dtype is not dt or v.dtype is not dt or (out is not None and out.dtype is not dt):
        raise ValueError(f"k / v / out dtype ({k.dtype}, {v.dtype}, {None if out is None else out.dtype}) "
                         f"differs from q's {dt}")
    if k.get_device() != dev or v.get_device() != dev or (out is not None and out.get_device() != dev):
        raise ValueError(f"k / v / out must be on q's device {q.device}")
    if out is not None and out.shape != qs:
        raise ValueError(f"out {tuple(out.shape)} must have q's shape {tuple(qs)}")
    if lse is not None:
        if lse.dtype is not torch.float32 or lse.get_device() != dev or not lse.is_contiguous():
            raise ValueError("lse must be a contiguous float32 tensor on q's device")
        if tuple(lse.shape) != tuple(lse_shape):
            raise ValueError(f"lse must have shape {tuple(lse_shape)} (got {tuple(lse.shape)})")


def _problem(q, k, *, scale, causal, window, alibi_slopes, softcap, q_pos_offset, kv_pos_offset,
             seqlen_kv_total) -> AttnProblem:
    B, Hq, Sq, D = q.shape
    Bk, Hkv, Skv, Dk = k.shape
    if Bk != B or Dk != D:
        raise ValueError("q and k disagree on batch or head_dim")
    if q.dtype not in _DT:
        raise ValueError(f"unsupported dtype {q.dtype}")
    if alibi_slopes is not None:
        if alibi_slopes.dtype != torch.float32 or alibi_slopes.device != q.device or alibi_slopes.numel() != Hq:
            raise ValueError("alibi_slopes must be a float32 tensor [Hq] on q's device")
    return AttnProblem(
        batch=B, heads_q=Hq, heads_kv=Hkv, seqlen_q=Sq, seqlen_kv=Skv, head_dim=D, dtype=_DT[q.dtype],
        scale=float(1.0 / math.sqrt(D) if scale is None else scale), softcap=float(softcap),
        alibi_slopes=None if alibi_slopes is None else alibi_slopes.data_ptr(), causal=int(bool(causal)),
        window_left=int(window[0]), window_right=int(window[1]),
        seqlen_kv_total=int(seqlen_kv_total or 0),
        q_pos_offset=_ffi.ATTN_Q_POS_DEFAULT if q_pos_offset is None else int(q_pos_offset),
        kv_pos_offset=int(kv_pos_offset))


def last_launch_count() -> int:
    """Kernels enqueued by the last successful call on this thread."""
    return load().attn_last_launch_count()


class repair_counters:
    """Context manager around ``attn_debug_repair_counters``: while active, the
    kernels count the warps that apply the Eq. 7 O-rescale into a
    device uint32 tensor of ``ATTN_REPAIR_SLOTS`` slots (test instrumentation).
    ``counts()`` reads them: a dict kernel name -> events."""

    NAMES = ("fwd128", "fwd64", "persist", "decode")

    def __init__(self, device="cuda"):
        self.buf = torch.zeros(_ffi.ATTN_REPAIR_SLOTS, dtype=torch.int32, device=device)

    def __enter__(self):
        load().attn_debug_repair_counters(self.buf.data_ptr())
        return self

    def __exit__(self, *exc):
        load().attn_debug_repair_counters(None)
        return False

    def counts(self) -> dict:
        torch.cuda.synchronize(self.buf.device)
        return dict(zip(self.NAMES, (int(x) for x in self.buf.cpu())))


def fused_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, scale: Optional[float] = None,
              causal: bool = False, window: Tuple[int, int] = (-1, -1),
              alibi_slopes: Optional[torch.Tensor] = None, softcap: float = 0.0,
              q_pos_offset: Optional[int] = None, kv_pos_offset: int = 0,
              seqlen_kv_total: Optional[int] = None, out: Optional[torch.Tensor] = None,
              lse: Optional[torch.Tensor] = None, return_lse: bool = False, kv_splits: int = 0, stream=None):
    """Rolling Update forward (``attn_fused_fwd`` / ``attn_fused_fwd_splitkv``).

    Device tensors run in place on ``stream``.  Host (CPU) tensors take the
    end-to-end path: copied to the current device, computed, copied back
    (pinned host memory makes the copies asynchronous).  ``kv_splits``: 0 lets
    the library split the KV axis across CTAs for small grids (NEXT-2), 1 never
    splits, n > 1 forces n splits."""
    lib = load()
    if q.device.type == "cpu":
        return _fused_fwd_host(q, k, v, out=out, return_lse=return_lse, kv_splits=kv_splits,
                               kw=dict(scale=scale, causal=causal, window=window, alibi_slopes=alibi_slopes,
                                       softcap=softcap, q_pos_offset=q_pos_offset, kv_pos_offset=kv_pos_offset,
                                       seqlen_kv_total=seqlen_kv_total))
    prob = _problem(q, k, scale=scale, causal=causal, window=window, alibi_slopes=alibi_slopes, softcap=softcap,
                    q_pos_offset=q_pos_offset, kv_pos_offset=kv_pos_offset, seqlen_kv_total=seqlen_kv_total)
    if out is None:
        out = torch.empty_like(q, memory_format=torch.contiguous_format)
    if return_lse and lse is None:
        lse = torch.empty(q.shape[:3], device=q.device, dtype=torch.float32)
    _check_io(q, k, v, out, lse, q.shape[:3])
    splits = kv_splits if kv_splits > 0 else lib.attn_fused_fwd_default_splits(ctypes.byref(prob), 0)
    if splits <= 1:
        check(lib.attn_fused_fwd(ctypes.byref(prob), _as_tensor(q), _as_tensor(k), _as_tensor(v), _as_tensor(out),
                                 None if lse is None else lse.data_ptr(), _stream(stream)), "attn_fused_fwd")
    else:
        need = lib.attn_fused_fwd_workspace_bytes(ctypes.byref(prob), splits)
        ws = _scratch(q.device, need, stream)
        check(lib.attn_fused_fwd_splitkv(ctypes.byref(prob), _as_tensor(q), _as_tensor(k), _as_tensor(v),
                                         _as_tensor(out), None if lse is None else lse.data_ptr(), splits,
                                         ws.data_ptr(), ws.numel(), _stream(stream)), "attn_fused_fwd_splitkv")
    return (out, lse) if return_lse else out


def fused_fwd_partial(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, scale: Optional[float] = None,
                      causal: bool = False, window: Tuple[int, int] = (-1, -1),
                      alibi_slopes: Optional[torch.Tensor] = None, softcap: float = 0.0,
                      q_pos_offset: Optional[int] = None, kv_pos_offset: int = 0,
                      seqlen_kv_total: Optional[int] = None, out: Optional[torch.Tensor] = None,
                      lse: Optional[torch.Tensor] = None, stream=None):
    """Rolling Update over a KV shard kept as an fp32 normalised partial
    (``attn_fused_fwd_partial``): returns (O_r fp32 [B, Hq, Sq, D], lse_r fp32 [B, Hq, Sq]),
    merged across shards by :func:`merge_partials` (context-parallel prefill)."""
    lib = load()
    prob = _problem(q, k, scale=scale, causal=causal, window=window, alibi_slopes=alibi_slopes, softcap=softcap,
                    q_pos_offset=q_pos_offset, kv_pos_offset=kv_pos_offset, seqlen_kv_total=seqlen_kv_total)
    if out is None:
        out = torch.empty(q.shape, dtype=torch.float32, device=q.device)
    if lse is None:
        lse = torch.empty(q.shape[:3], dtype=torch.float32, device=q.device)
    _check_io(q, k, v, None, lse, q.shape[:3])
    if out.dtype != torch.float32 or tuple(out.shape) != tuple(q.shape) or not out.is_contiguous() \
            or out.device != q.device:
        raise ValueError("out must be a contiguous float32 tensor of q's shape")
    check(lib.attn_fused_fwd_partial(ctypes.byref(prob), _as_tensor(q), _as_tensor(k), _as_tensor(v), out.data_ptr(),
                                     lse.data_ptr(), _stream(stream)), "attn_fused_fwd_partial")
    return out, lse


_SCRATCH = {}


def _torch_stream(device, stream):
    return torch.cuda.current_stream(device) if stream is None else stream


def _scratch(device, need: int, stream) -> torch.Tensor:
    """Per-(device, stream) scratch for the split-KV prefill partials (no zeroing needed).
    Allocated ON the stream that uses it, so when a larger one replaces it the caching
    allocator recycles the old block in that stream's order (never under a running kernel)."""
    st = _torch_stream(device, stream)
    key = (device.index if device.index is not None else torch.cuda.current_device(), st.cuda_stream)
    ws = _SCRATCH.get(key)
    if ws is None or ws.numel() < need:
        with torch.cuda.stream(st):
            ws = torch.empty(max(need, 1 << 20), dtype=torch.uint8, device=device)
        _SCRATCH[key] = ws
    return ws


_HOST_STREAMS = {}


def _fused_fwd_host(q, k, v, *, out, return_lse, kv_splits, kw, chunks: int = 8):
    """End-to-end call on HOST tensors: the batch is cut into chunks that flow through two
    CUDA streams, so the host->device copy of chunk c+1 overlaps the kernel and the
    device->host copy of chunk c (pinned host memory makes the copies asynchronous).
    Returns when the result is in host memory."""
    dev = torch.device("cuda", torch.cuda.current_device())
    streams = _HOST_STREAMS.get(dev.index)
    if streams is None:
        streams = _HOST_STREAMS[dev.index] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    B = q.shape[0]
    n = max(1, min(chunks, B))
    bounds = [B * i // n for i in range(n + 1)]
    pin = q.is_pinned()
    if out is None:
        out = torch.empty(q.shape, dtype=q.dtype, pin_memory=pin)
    lse = torch.empty(q.shape[:3], dtype=torch.float32, pin_memory=pin) if return_lse else None
    cur = torch.cuda.current_stream(dev)
    sl = kw.pop("alibi_slopes")
    for st in streams:
        st.wait_stream(cur)
    for c in range(n):
        st = streams[c % 2]
        b0, b1 = bounds[c], bounds[c + 1]
        with torch.cuda.stream(st):
            qd, kd, vd = (t[b0:b1].to(dev, non_blocking=True) for t in (q, k, v))
            sld = None if sl is None else sl.to(dev, non_blocking=True)
            res = fused_fwd(qd, kd, vd, alibi_slopes=sld, return_lse=return_lse, kv_splits=kv_splits,
                            stream=st, **kw)
            o_d, l_d = res if return_lse else (res, None)
            out[b0:b1].copy_(o_d, non_blocking=True)
            if lse is not None:
                lse[b0:b1].copy_(l_d, non_blocking=True)
    for st in streams:
        st.synchronize()
    return (out, lse) if return_lse else out


class Parts:
    """Partial (m, l, O) triples of Split-K Update (Fig. 5): m, l [P, B, H]
    and o [P, B, H, D] fp32 views (any strides with a contiguous D)."""

    def __init__(self, m: torch.Tensor, l: torch.Tensor, o: torch.Tensor):
        if m.stride() != l.stride():
            raise ValueError("m and l must share strides")
        if o.stride(3) != 1:
            raise ValueError("o must be contiguous over D")
        self.m, self.l, self.o = m, l, o

    @staticmethod
    def empty(P: int, B: int, H: int, D: int, device) -> "Parts":
        return Parts(torch.empty(P, B, H, device=device), torch.empty(P, B, H, device=device),
                     torch.empty(P, B, H, D, device=device))

    @staticmethod
    def packed(buf: torch.Tensor) -> "Parts":
        """Views over one [P, B, H, D + 2] fp32 buffer: O at [..., :D], m at D, l at D + 1
        (the all-gather layout of the KV-sharded decode)."""
        D = buf.shape[-1] - 2
        return Parts(buf[..., D], buf[..., D + 1], buf[..., :D])

    def c(self) -> AttnParts:
        m, o = self.m, self.o
        return AttnParts(m.data_ptr(), self.l.data_ptr(), o.data_ptr(), m.shape[0], m.stride(0), m.stride(1),
                         m.stride(2), o.stride(0), o.stride(1), o.stride(2))


def default_splits(q: torch.Tensor, k: torch.Tensor, sm_count: int = 0) -> int:
    prob = _problem(q, k, scale=None, causal=False, window=(-1, -1), alibi_slopes=None, softcap=0.0,
                    q_pos_offset=None, kv_pos_offset=0, seqlen_kv_total=None)
    return load().attn_splitkv_default_splits(ctypes.byref(prob), sm_count)


def workspace_bytes(q: torch.Tensor, k: torch.Tensor, num_splits: int = 0) -> int:
    prob = _problem(q, k, scale=None, causal=False, window=(-1, -1), alibi_slopes=None, softcap=0.0,
                    q_pos_offset=None, kv_pos_offset=0, seqlen_kv_total=None)
    return load().attn_splitkv_workspace_bytes(ctypes.byref(prob), num_splits)


_WS_CACHE = {}


def _decode_workspace(device, need: int, ticket_bytes: int, stream) -> torch.Tensor:
    """Per-(device, stream) decode workspace.  Its leading ticket block must be zero
    before a call and every call leaves it zero (include/attn.h), so only a ticket
    block larger than any before it (which may overlap old partials) is cleared."""
    st = _torch_stream(device, stream)
    key = (device.index if device.index is not None else torch.cuda.current_device(), st.cuda_stream)
    ws, clean = _WS_CACHE.get(key, (None, 0))
    with torch.cuda.stream(st):   # allocated and zeroed in the order of the stream that uses it
        if ws is None or ws.numel() < need:
            ws = torch.zeros(max(need, 1 << 20), dtype=torch.uint8, device=device)
            clean = ws.numel()
        if ticket_bytes > clean:
            ws[:ticket_bytes].zero_()
    _WS_CACHE[key] = (ws, ticket_bytes)   # after the call: tickets zero, partials beyond dirty
    return ws


def splitkv_decode(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, num_splits: int = 0,
                   scale: Optional[float] = None, causal: bool = False, window: Tuple[int, int] = (-1, -1),
                   alibi_slopes: Optional[torch.Tensor] = None, softcap: float = 0.0,
                   q_pos_offset: Optional[int] = None, kv_pos_offset: int = 0,
                   seqlen_kv_total: Optional[int] = None, out: Optional[torch.Tensor] = None,
                   lse: Optional[torch.Tensor] = None, return_lse: bool = False, parts: Optional[Parts] = None,
                   workspace: Optional[torch.Tensor] = None, want_out: bool = True,
                   packed: Optional[torch.Tensor] = None, stream=None):
    """Split-K Update decode (``attn_splitkv_decode``): q [B, Hq, Sq, D] bf16/fp16 with
    Sq = 1, or a few query tokens (multi-token decode) with G * Sq <= 16 packed rows.

    ``parts`` receives the raw local-section triples; with ``want_out`` the
    Eq. 8 combine also produces O (and lse) -- fused into the split kernel
    when ``parts`` is None.  ``packed`` (fp32 [B, Hq, D + 2], Sq = 1): the fused
    combine writes the UN-normalised merged triple there instead
    (``attn_splitkv_decode_packed``; returns ``packed``).  A caller-supplied
    ``workspace`` must be zeroed before its first use (its ticket block;
    include/attn.h)."""
    lib = load()
    if q.device.type == "cpu":
        dev = torch.device("cuda", torch.cuda.current_device())
        qd, kd, vd = (t.to(dev, non_blocking=True) for t in (q, k, v))
        sl = None if alibi_slopes is None else alibi_slopes.to(dev, non_blocking=True)
        res = splitkv_decode(qd, kd, vd, num_splits=num_splits, scale=scale, causal=causal, window=window,
                             alibi_slopes=sl, softcap=softcap, q_pos_offset=q_pos_offset,
                             kv_pos_offset=kv_pos_offset, seqlen_kv_total=seqlen_kv_total, return_lse=return_lse,
                             stream=stream)
        if return_lse:
            return res[0].cpu(), res[1].cpu()
        return res.cpu()
    prob = _problem(q, k, scale=scale, causal=causal, window=window, alibi_slopes=alibi_slopes, softcap=softcap,
                    q_pos_offset=q_pos_offset, kv_pos_offset=kv_pos_offset, seqlen_kv_total=seqlen_kv_total)
    if num_splits == 0:
        num_splits = lib.attn_splitkv_default_splits(ctypes.byref(prob), 0)
    if packed is not None:
        B, Hq, Sq, D = q.shape
        _check_io(q, k, v)
        if Sq != 1 or packed.dtype != torch.float32 or tuple(packed.shape) != (B, Hq, D + 2) \
                or not packed.is_contiguous() or packed.device != q.device:
            raise ValueError(f"packed must be a contiguous float32 [{B}, {Hq}, {D + 2}] tensor (Sq = 1)")
        need = lib.attn_splitkv_workspace_bytes(ctypes.byref(prob), num_splits)
        if workspace is None:
            workspace = _decode_workspace(q.device, need, (B * k.shape[1] * 4 + 255) // 256 * 256, stream)
        elif workspace.numel() * workspace.element_size() < need or workspace.device != q.device:
            raise ValueError(f"workspace must be >= {need} bytes on q's device")
        check(lib.attn_splitkv_decode_packed(ctypes.byref(prob), _as_tensor(q), _as_tensor(k), _as_tensor(v),
                                             num_splits, workspace.data_ptr(),
                                             workspace.numel() * workspace.element_size(), packed.data_ptr(),
                                             _stream(stream)), "attn_splitkv_decode_packed")
        return packed
    if want_out and out is None:
        out = torch.empty_like(q, memory_format=torch.contiguous_format)
    if not want_out:
        out = None
    lse_shape = q.shape[:2] if q.shape[2] == 1 else q.shape[:3]   # [B, Hq] for one query, else [B, Hq, Sq]
    if return_lse and lse is None and want_out:
        lse = torch.empty(lse_shape, device=q.device, dtype=torch.float32)
    _check_io(q, k, v, out, lse, lse_shape)
    if parts is not None:
        P, B, H, D = parts.o.shape
        if (P, B, H, D) != (num_splits, q.shape[0], q.shape[1], q.shape[3]) or parts.m.shape != (P, B, H) \
                or parts.l.shape != (P, B, H) or any(t.dtype != torch.float32 or t.device != q.device
                                                     for t in (parts.m, parts.l, parts.o)):
            raise ValueError(f"parts must be float32 [{num_splits}, B, Hq(, D)] triples on q's device")
    ws_ptr, ws_bytes = None, 0
    if parts is None:
        need = lib.attn_splitkv_workspace_bytes(ctypes.byref(prob), num_splits)
        if workspace is None:
            tb = (q.shape[0] * k.shape[1] * 4 + 255) // 256 * 256
            workspace = _decode_workspace(q.device, need, tb, stream)
        elif workspace.numel() * workspace.element_size() < need or workspace.device != q.device:
            raise ValueError(f"workspace must be >= {need} bytes on q's device "
                             f"(attn_splitkv_workspace_bytes); got {workspace.numel() * workspace.element_size()}")
        ws_ptr, ws_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    cparts = None if parts is None else ctypes.byref(parts.c())
    check(lib.attn_splitkv_decode(ctypes.byref(prob), _as_tensor(q), _as_tensor(k), _as_tensor(v), num_splits,
                                  ws_ptr, ws_bytes, cparts, _as_tensor(out), None if lse is None else lse.data_ptr(),
                                  _stream(stream)), "attn_splitkv_decode")
    if not want_out:
        return parts
    return (out, lse) if return_lse else out


def combine(parts: Parts, *, out: Optional[torch.Tensor] = None, out_dtype=torch.bfloat16,
            lse: Optional[torch.Tensor] = None, return_lse: bool = False, acc: Optional[Parts] = None,
            want_out: bool = True, stream=None):
    """Split-K global section (``attn_combine``, Eq. 8) over parts [P, B, H(, D)].

    ``out`` gets O / L as [B, H, 1, D]; ``acc`` (num_parts = 1) gets the
    un-normalised merged triple for a further hierarchical merge."""
    lib = load()
    P, B, H, D = parts.o.shape
    if want_out and out is None:
        out = torch.empty(B, H, 1, D, device=parts.o.device, dtype=out_dtype)
    if not want_out:
        out = None
    if return_lse and lse is None:
        lse = torch.empty(B, H, device=parts.o.device, dtype=torch.float32)
    for t in (parts.m, parts.l, parts.o):
        if t.dtype != torch.float32 or t.device != parts.o.device:
            raise ValueError("parts must be float32 tensors on one device")
    if parts.m.shape != (P, B, H) or parts.l.shape != (P, B, H):
        raise ValueError("parts m / l must be [P, B, H]")
    if out is not None and (tuple(out.shape) != (B, H, 1, D) or out.dtype not in _DT or out.device != parts.o.device):
        raise ValueError(f"out must be a [{B}, {H}, 1, {D}] tensor on the parts' device")
    if lse is not None and (tuple(lse.shape) != (B, H) or lse.dtype != torch.float32 or not lse.is_contiguous()
                            or lse.device != parts.o.device):
        raise ValueError(f"lse must be a contiguous float32 [{B}, {H}] tensor")
    if acc is not None and (acc.o.shape != (1, B, H, D) or acc.m.shape != (1, B, H) or acc.o.dtype != torch.float32):
        raise ValueError(f"acc must be float32 [1, {B}, {H}(, {D})] triples")
    dt = _DT[out.dtype] if out is not None else _ffi.ATTN_FP32
    cacc = None if acc is None else ctypes.byref(acc.c())
    check(lib.attn_combine(B, H, D, ctypes.byref(parts.c()), dt, _as_tensor(out),
                           None if lse is None else lse.data_ptr(), cacc, _stream(stream)), "attn_combine")
    if return_lse:
        return out, lse
    return out


def merge_partials(o_parts: torch.Tensor, lse_parts: torch.Tensor, *, out: Optional[torch.Tensor] = None,
                   out_dtype=None, return_lse: bool = False, stream=None):
    """Eq. 8 over P normalised partials (``attn_merge_partials``):
    o_parts [P, ..., D] (bf16/fp16/fp32), lse_parts [P, ...] fp32, with the
    middle dimensions flattened into rows.  Returns O [..., D] (and lse)."""
    lib = load()
    if o_parts.dtype not in _DT or lse_parts.dtype != torch.float32 or lse_parts.device != o_parts.device:
        raise ValueError("o_parts must be bf16/fp16/fp32 and lse_parts float32 on the same device")
    if tuple(lse_parts.shape) != tuple(o_parts.shape[:-1]):
        raise ValueError(f"lse_parts {tuple(lse_parts.shape)} must be o_parts' shape without D")
    P, D = o_parts.shape[0], o_parts.shape[-1]
    rows = lse_parts[0].numel()
    o2 = o_parts.reshape(P, rows, D)
    l2 = lse_parts.reshape(P, rows)
    if o2.stride(2) != 1 or l2.stride(1) != 1:
        raise ValueError("partials must be contiguous over D and rows")
    dt = o_parts.dtype if out_dtype is None else out_dtype
    if out is None:
        out = torch.empty(o_parts.shape[1:], dtype=dt, device=o_parts.device)
    elif tuple(out.shape) != tuple(o_parts.shape[1:]) or out.dtype not in _DT or out.device != o_parts.device \
            or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous {tuple(o_parts.shape[1:])} tensor on the parts' device")
    lse = torch.empty(lse_parts.shape[1:], dtype=torch.float32, device=o_parts.device) if return_lse else None
    out2 = out.view(rows, D)
    check(lib.attn_merge_partials(P, rows, D, _DT[o_parts.dtype], o2.data_ptr(), o2.stride(0), o2.stride(1),
                                  l2.data_ptr(), l2.stride(0), _DT[out.dtype], out2.data_ptr(), out2.stride(0),
                                  None if lse is None else lse.data_ptr(), _stream(stream)), "attn_merge_partials")
    return (out, lse) if return_lse else out


def softmax_rows(x: torch.Tensor, *, out: Optional[torch.Tensor] = None, want_out: bool = True,
                 return_stats: bool = False, stream=None):
    """The Fig. 2 reduction chain (``attn_softmax_rows``) on a [rows, cols] tensor:
    softmax y, and with ``return_stats`` the row max and Fig. 2a's row sum
    sum exp(x - max)."""
    lib = load()
    if x.dim() != 2 or x.stride(1) != 1:
        raise ValueError("x must be [rows, cols] with contiguous columns")
    rows, cols = x.shape
    y = None
    if want_out:
        if out is None:   # rows padded to a 16-byte multiple (the kernel's vector alignment)
            per16 = 16 // x.element_size()
            y = torch.empty(rows, -(-cols // per16) * per16, dtype=x.dtype, device=x.device)[:, :cols]
        else:
            y = out
    m = torch.empty(rows, device=x.device, dtype=torch.float32) if return_stats else None
    l = torch.empty(rows, device=x.device, dtype=torch.float32) if return_stats else None
    check(lib.attn_softmax_rows(rows, cols, _DT[x.dtype], x.data_ptr(), x.stride(0),
                                None if y is None else y.data_ptr(), 0 if y is None else y.stride(0),
                                None if m is None else m.data_ptr(), None if l is None else l.data_ptr(),
                                _stream(stream)), "attn_softmax_rows")
    if return_stats:
        return y, m, l
    return y
