"""Multi-GPU partitioning of the hot path (one process per GPU, torch.distributed).

* Prefill (Rolling Update) shards independent (b, h) units: nothing is
  exchanged (``shard_range``).
* Long-context decode shards the KV sequence (``decode_kv_sharded``): each
  rank runs the Split-K local section over its keys
  [r L / W, (r + 1) L / W) with ``kv_pos_offset`` set to the shard start,
  merges its splits into ONE un-normalised (m, l, O) triple per (b, h)
  (Eq. 8 without the divide), all-gathers the packed [B, H, D + 2] fp32
  triples (the only collective on the path), and applies the Eq. 8 combine
  over the W parts.  Exact because h commutes with the reducer (Eq. 4,
  P:578-579), so the merge may be grouped by split and then by rank.

* Long-context prefill (context parallel, NEXT-3) shards the KV sequence the
  same way (``prefill_kv_sharded``): every rank runs the Rolling Update kernel
  on its keys with absolute positions, the normalised (O_r, lse_r) pairs are
  all-gathered and merged with Eq. 8 (``attn_merge_partials``).

The local section and the combine are injectable so the host-side logic can
be tested on CPU with world_size 2 over gloo; the defaults are the CUDA
kernels behind the C ABI.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist

from . import Parts, combine, splitkv_decode


def shard_range(n: int, rank: int, world: int):
    """Contiguous, balanced [lo, hi) of n units for `rank` (first n % W ranks get one more)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _local_kernels(q, k_shard, v_shard, *, kv_pos_offset, seqlen_kv_total, num_splits, variant):
    B, Hq, _, D = q.shape
    splits = num_splits
    if splits == 0:
        from . import default_splits
        splits = default_splits(q, k_shard)
    parts = Parts.empty(splits, B, Hq, D, q.device)
    splitkv_decode(q, k_shard, v_shard, num_splits=splits, parts=parts, want_out=False,
                   kv_pos_offset=kv_pos_offset, seqlen_kv_total=seqlen_kv_total, **variant)
    return parts


def _merge_kernels(parts: Parts, acc: Parts):
    combine(parts, acc=acc, want_out=False)


def _final_kernels(parts: Parts, out_dtype, return_lse):
    return combine(parts, out_dtype=out_dtype, return_lse=return_lse)


def decode_kv_sharded(q: torch.Tensor, k_shard: torch.Tensor, v_shard: torch.Tensor, *, kv_pos_offset: int,
                      seqlen_kv_total: int, group=None, num_splits: int = 0, return_lse: bool = False,
                      local: Optional[Callable] = None, merge: Optional[Callable] = None,
                      final: Optional[Callable] = None, **variant):
    """KV-sequence-sharded Split-K decode. q [B, Hq, 1, D] is replicated;
    k_shard/v_shard [B, Hkv, L_r, D] hold keys [kv_pos_offset, kv_pos_offset + L_r)
    of a sequence of seqlen_kv_total keys.  Returns O [B, Hq, 1, D] (and lse)
    on every rank."""
    final = final or _final_kernels
    world = dist.get_world_size(group)
    B, Hq, _, D = q.shape
    send = torch.empty(1, B, Hq, D + 2, dtype=torch.float32, device=q.device)
    if local is None and merge is None:
        # one launch: the split kernel's fused Eq. 8 section writes this rank's merged,
        # un-normalised triples straight into the send buffer
        splitkv_decode(q, k_shard, v_shard, num_splits=num_splits, packed=send[0], kv_pos_offset=kv_pos_offset,
                       seqlen_kv_total=seqlen_kv_total, **variant)
    else:
        local = local or _local_kernels
        merge = merge or _merge_kernels
        parts = local(q, k_shard, v_shard, kv_pos_offset=kv_pos_offset, seqlen_kv_total=seqlen_kv_total,
                      num_splits=num_splits, variant=variant)
        merge(parts, Parts.packed(send))
    recv = torch.empty(world, B, Hq, D + 2, dtype=torch.float32, device=q.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    return final(Parts.packed(recv), q.dtype, return_lse)


# ----------------------------------------------------------------------------- context-parallel prefill (NEXT-3)
def _prefill_local(q, k_shard, v_shard, *, kv_pos_offset, seqlen_kv_total, variant):
    from . import fused_fwd_partial
    # fp32 normalised partial: the gathered (O_r, lse_r) carry no 16-bit rounding into Eq. 8
    return fused_fwd_partial(q, k_shard, v_shard, kv_pos_offset=kv_pos_offset, seqlen_kv_total=seqlen_kv_total,
                             **variant)


def prefill_kv_sharded(q: torch.Tensor, k_shard: torch.Tensor, v_shard: torch.Tensor, *, kv_pos_offset: int,
                       seqlen_kv_total: int, group=None, out_dtype=None, local: Optional[Callable] = None,
                       final: Optional[Callable] = None, **variant):
    """Context-parallel (KV-sharded) Rolling Update prefill: every rank holds all
    queries and keys [kv_pos_offset, kv_pos_offset + L_r) of a sequence of
    seqlen_kv_total keys.  Each rank runs the fused forward on its shard (the
    mask uses absolute positions), the (O_r, lse_r) pairs are all-gathered and
    merged with the Eq. 8 combine (the paper's rolling update composed with
    privatisation, Fig. 19, lifted to GPUs).  Returns O [B, H, Sq, D] (and lse
    [B, H, Sq]) on every rank."""
    local = local or _prefill_local
    world = dist.get_world_size(group)
    B, H, S, D = q.shape
    o_r, lse_r = local(q, k_shard, v_shard, kv_pos_offset=kv_pos_offset, seqlen_kv_total=seqlen_kv_total,
                       variant=variant)
    # gathered along dim 0 ([W*B, ...]; gloo requires it), then viewed as [W, B, ...]
    o_all = torch.empty((world * B,) + tuple(o_r.shape[1:]), dtype=o_r.dtype, device=o_r.device)
    lse_all = torch.empty((world * B,) + tuple(lse_r.shape[1:]), dtype=lse_r.dtype, device=o_r.device)
    dist.all_gather_into_tensor(o_all, o_r.contiguous(), group=group)
    dist.all_gather_into_tensor(lse_all, lse_r.contiguous(), group=group)
    o_all = o_all.view((world,) + tuple(o_r.shape))
    lse_all = lse_all.view((world,) + tuple(lse_r.shape))
    return merge_prefill_parts(o_all, lse_all, out_dtype or q.dtype, final=final)


def merge_prefill_parts(o_all: torch.Tensor, lse_all: torch.Tensor, out_dtype, final: Optional[Callable] = None):
    """Eq. 8 over W normalised partials o_all [W, B, H, S, D], lse_all [W, B, H, S]
    (a normalised (O, lse) is the repaired triple (m = lse, l = 1, O))."""
    if final is not None:
        return final(o_all, lse_all, out_dtype)
    from . import merge_partials
    return merge_partials(o_all, lse_all, out_dtype=out_dtype, return_lse=True)


class NcclComm:
    """A communicator of the C ABI's own NCCL path (``attn_nccl_comm_init``): the
    whole KV-sharded decode step -- local section, local merge, all-gather, Eq. 8 --
    is ONE library call (``attn_decode_kv_sharded``) with no torch on the data path.
    The 128-byte unique id is created on rank 0 and shipped out of band, here
    through an existing torch.distributed group (any backend) when given."""

    def __init__(self, rank: int, world: int, unique_id: Optional[bytes] = None, group=None):
        import ctypes
        from ._ffi import check, load
        lib = load()
        if unique_id is None:
            buf = ctypes.create_string_buffer(128)
            if rank == 0:
                check(lib.attn_nccl_get_unique_id(buf), "attn_nccl_get_unique_id")
            if world > 1:
                obj = [buf.raw if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0, group=group)
                buf = ctypes.create_string_buffer(obj[0], 128)
            unique_id = buf.raw
        self._h = ctypes.c_void_p()
        check(lib.attn_nccl_comm_init(ctypes.byref(self._h), world, rank, ctypes.create_string_buffer(unique_id, 128)),
              "attn_nccl_comm_init")
        self.rank, self.world = rank, world

    @staticmethod
    def unique_id() -> bytes:
        import ctypes
        from ._ffi import check, load
        buf = ctypes.create_string_buffer(128)
        check(load().attn_nccl_get_unique_id(buf), "attn_nccl_get_unique_id")
        return buf.raw

    def close(self):
        from ._ffi import check, load
        if self._h:
            check(load().attn_nccl_comm_destroy(self._h), "attn_nccl_comm_destroy")
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def decode_kv_sharded(self, q: torch.Tensor, k_shard: torch.Tensor, v_shard: torch.Tensor, *,
                          kv_pos_offset: int, seqlen_kv_total: int, out: Optional[torch.Tensor] = None,
                          return_lse: bool = False, workspace: Optional[torch.Tensor] = None, stream=None,
                          **variant):
        """``attn_decode_kv_sharded`` on this communicator (same contract as
        :func:`decode_kv_sharded`; identical O, lse on every rank).  A caller-supplied
        ``workspace`` must be zeroed before its first use (include/attn.h)."""
        import ctypes
        from . import _as_tensor, _problem, _stream
        from ._ffi import check, load
        lib = load()
        prob = _problem(q, k_shard, scale=variant.get("scale"), causal=variant.get("causal", False),
                        window=variant.get("window", (-1, -1)), alibi_slopes=variant.get("alibi_slopes"),
                        softcap=variant.get("softcap", 0.0), q_pos_offset=variant.get("q_pos_offset"),
                        kv_pos_offset=kv_pos_offset, seqlen_kv_total=seqlen_kv_total)
        from . import _check_io, _torch_stream
        need = lib.attn_decode_kv_sharded_workspace_bytes(ctypes.byref(prob), self.world)
        if workspace is None:   # cached per communicator; zeroed once (its ticket block), left zero by every call
            ws = getattr(self, "_ws", None)
            if ws is None or ws.numel() < need or ws.device != q.device:
                with torch.cuda.stream(_torch_stream(q.device, stream)):
                    self._ws = torch.zeros(need, dtype=torch.uint8, device=q.device)
            workspace = self._ws
        elif workspace.numel() * workspace.element_size() < need or workspace.device != q.device:
            raise ValueError(f"workspace must be >= {need} bytes on q's device (zeroed before first use)")
        if out is None:
            out = torch.empty_like(q, memory_format=torch.contiguous_format)
        lse = torch.empty(q.shape[:2], device=q.device, dtype=torch.float32) if return_lse else None
        _check_io(q, k_shard, v_shard, out, lse, q.shape[:2])
        check(lib.attn_decode_kv_sharded(self._h, ctypes.byref(prob), _as_tensor(q), _as_tensor(k_shard),
                                         _as_tensor(v_shard), workspace.data_ptr(),
                                         workspace.numel() * workspace.element_size(), _as_tensor(out),
                                         None if lse is None else lse.data_ptr(), _stream(stream)),
              "attn_decode_kv_sharded")
        return (out, lse) if return_lse else out
