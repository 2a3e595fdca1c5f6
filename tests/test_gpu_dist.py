"""GPU coverage of the KV-sharded decode (paper_2510_08726_b200.dist) on one
GPU: W shards are run one after the other through the same local/merge/final
steps decode_kv_sharded uses, the "all-gather" is a loopback copy into the
packed [W, B, H, D+2] buffer, and the result must equal the unsharded oracle.
A real 1-rank NCCL process group also runs decode_kv_sharded end to end."""
import math
import os

import numpy as np
import pytest
import torch

import datagen
import oracle
from datagen import device as dgd
from tests.helpers import LSE_TOL_BF16, assert_bf16_close, assert_lse_close, gen_qkv, problem

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import torch.distributed as dist

    import paper_2510_08726_b200 as pb
    from paper_2510_08726_b200 import dist as pdist


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("W", [2, 3, 8])
def test_kv_sharded_decode_loopback(W, fused):
    """fused: each shard's split kernel writes its merged un-normalised triple straight into
    the packed send slot (attn_splitkv_decode_packed, one launch); else raw split triples +
    a separate attn_combine(acc_out).  Each shard's packed (m, l) must give the oracle's lse
    over the shard's keys; Eq. 8 over the W slots must give the unsharded oracle."""
    B, Hq, Hkv, L, D = 2, 8, 2, 3001, 128
    p = problem(B, Hq, Hkv, 1, L, D, causal=True)
    raw, f64 = gen_qkv(900 + W, B, Hq, Hkv, 1, L, D)
    ref_o, ref_l = oracle.attention(p, *f64)
    q, k, v = (dgd.to_device(x) for x in raw)
    packed = torch.empty(W, B, Hq, D + 2, device="cuda")
    for r in range(W):
        lo, hi = pdist.shard_range(L, r, W)
        ks, vs = k[:, :, lo:hi].contiguous(), v[:, :, lo:hi].contiguous()
        if fused:
            pb.splitkv_decode(q, ks, vs, packed=packed[r], kv_pos_offset=lo, seqlen_kv_total=L, causal=True)
            torch.cuda.synchronize()
            assert pb.last_launch_count() == 1
        else:
            parts = pdist._local_kernels(q, ks, vs, kv_pos_offset=lo, seqlen_kv_total=L, num_splits=0,
                                         variant=dict(causal=True))
            pdist._merge_kernels(parts, pb.Parts.packed(packed[r:r + 1]))
        ps = problem(B, Hq, Hkv, 1, hi - lo, D, causal=True, seqlen_kv_total=L, q_pos_offset=L - 1, kv_pos_offset=lo)
        _, rl = oracle.attention(ps, f64[0], f64[1][:, :, lo:hi], f64[2][:, :, lo:hi])
        pk = packed[r].cpu().numpy().astype(np.float64)
        assert_lse_close(pk[..., D] + np.log(pk[..., D + 1]), rl[:, :, 0], LSE_TOL_BF16, f"shard {r} (m, l)")
    out, lse = pdist._final_kernels(pb.Parts.packed(packed), torch.bfloat16, True)
    assert_bf16_close(out.float().cpu().numpy().astype(np.float64), ref_o, f"W={W}")
    assert_lse_close(lse.cpu().numpy(), ref_l[:, :, 0], LSE_TOL_BF16, "lse")


def test_kv_sharded_decode_nccl_one_rank():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(29700 + os.getpid() % 200))
    created = False
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        created = True
    try:
        B, Hq, Hkv, L, D = 1, 8, 2, 2048, 128
        p = problem(B, Hq, Hkv, 1, L, D, causal=True)
        raw, f64 = gen_qkv(77, B, Hq, Hkv, 1, L, D)
        ref_o, _ = oracle.attention(p, *f64)
        q, k, v = (dgd.to_device(x) for x in raw)
        out = pdist.decode_kv_sharded(q, k, v, kv_pos_offset=0, seqlen_kv_total=L, causal=True)
        assert_bf16_close(out.float().cpu().numpy().astype(np.float64), ref_o, "nccl 1 rank")
    finally:
        if created:
            dist.destroy_process_group()


@pytest.mark.parametrize("variant", [dict(causal=True), dict(causal=True, alibi=True), dict(softcap=2.0)])
def test_kv_sharded_decode_c_abi_one_rank(variant):
    """attn_nccl_comm_init + attn_decode_kv_sharded (the C ABI's own NCCL path, one call
    for local section + local merge + ncclAllGather + Eq. 8) on a 1-rank communicator;
    also a shard that is a suffix of a longer sequence (absolute positions)."""
    variant = dict(variant)
    B, Hq, Hkv, L, D = 2, 8, 2, 3001, 128
    alibi = variant.pop("alibi", False)
    p = problem(B, Hq, Hkv, 1, L, D, alibi_slopes=datagen.alibi_slopes(Hq) if alibi else None, **variant)
    raw, f64 = gen_qkv(1300, B, Hq, Hkv, 1, L, D)
    ref_o, ref_l = oracle.attention(p, *f64)
    q, k, v = (dgd.to_device(x) for x in raw)
    if alibi:
        variant["alibi_slopes"] = torch.tensor(datagen.alibi_slopes(Hq), dtype=torch.float32, device="cuda")
    comm = pdist.NcclComm(0, 1)
    try:
        out, lse = comm.decode_kv_sharded(q, k, v, kv_pos_offset=0, seqlen_kv_total=L, return_lse=True, **variant)
        torch.cuda.synchronize()
        assert pb.last_launch_count() == 2            # decode with fused local merge + final combine (+ NCCL)
        assert_bf16_close(out.float().cpu().numpy().astype(np.float64), ref_o, f"C-ABI kv-sharded {variant}")
        assert_lse_close(lse.cpu().numpy(), ref_l[:, :, 0], LSE_TOL_BF16, "C-ABI kv-sharded lse")
        # a shard holding keys [lo, L) of the sequence: the rank's part of the answer
        lo = 1000
        ps = problem(B, Hq, Hkv, 1, L - lo, D, seqlen_kv_total=L, q_pos_offset=L - 1, kv_pos_offset=lo,
                     alibi_slopes=p.alibi_slopes, **variant_no_slopes(variant))
        ref_s, _ = oracle.attention(ps, f64[0], f64[1][:, :, lo:], f64[2][:, :, lo:])
        out_s = comm.decode_kv_sharded(q, k[:, :, lo:].contiguous(), v[:, :, lo:].contiguous(), kv_pos_offset=lo,
                                       seqlen_kv_total=L, **variant)
        assert_bf16_close(out_s.float().cpu().numpy().astype(np.float64), ref_s, "C-ABI suffix shard")
        # the whole call (decode, NCCL all-gather, combine) captured in a CUDA graph and replayed
        out_g = torch.empty_like(q)
        ws = torch.zeros(pb.load().attn_decode_kv_sharded_workspace_bytes(
            __import__("ctypes").byref(pb._problem(q, k, scale=None, causal=p.causal, window=(-1, -1),
                                                   alibi_slopes=variant.get("alibi_slopes"), softcap=p.softcap,
                                                   q_pos_offset=None, kv_pos_offset=0, seqlen_kv_total=L)), 1),
            dtype=torch.uint8, device="cuda")
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            comm.decode_kv_sharded(q, k, v, kv_pos_offset=0, seqlen_kv_total=L, out=out_g, workspace=ws, **variant)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            comm.decode_kv_sharded(q, k, v, kv_pos_offset=0, seqlen_kv_total=L, out=out_g, workspace=ws, **variant)
        out_g.zero_()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out_g, out)
        assert int(ws[:256].count_nonzero()) == 0     # tickets reset by every replay
    finally:
        comm.close()


def variant_no_slopes(v):
    return {k: x for k, x in v.items() if k != "alibi_slopes"}


# --------------------------------------------------------------------------- context-parallel prefill (NEXT-3)
@pytest.mark.parametrize("W,variant,D", [(2, dict(causal=True), 128), (3, dict(causal=True, window_left=300), 128),
                                         (4, dict(), 128), (3, dict(causal=True), 64)])
def test_kv_sharded_prefill_loopback(W, variant, D):
    """Context-parallel prefill: every shard's fp32 normalised partial (attn_fused_fwd_partial)
    equals the oracle restricted to the shard's keys (absolute positions), and Eq. 8 over
    the shards equals the oracle over all keys."""
    B, Hq, Hkv, S = 1, 4, 2, 700
    kw = dict(variant)
    p = problem(B, Hq, Hkv, S, S, D, **kw)
    raw, f64 = gen_qkv(1200 + W, B, Hq, Hkv, S, S, D)
    ref_o, ref_l = oracle.attention(p, *f64)
    q, k, v = (dgd.to_device(x) for x in raw)
    win = (kw.pop("window_left", -1), -1)
    o_all = torch.empty(W, B, Hq, S, D, dtype=torch.float32, device="cuda")
    lse_all = torch.empty(W, B, Hq, S, device="cuda")
    for r in range(W):
        lo, hi = pdist.shard_range(S, r, W)
        o_r, l_r = pdist._prefill_local(q, k[:, :, lo:hi].contiguous(), v[:, :, lo:hi].contiguous(),
                                        kv_pos_offset=lo, seqlen_kv_total=S, variant=dict(window=win, **kw))
        assert o_r.dtype == torch.float32
        pr = problem(B, Hq, Hkv, S, hi - lo, D, kv_pos_offset=lo, seqlen_kv_total=S, q_pos_offset=0,
                     window_left=win[0], **kw)
        ro, rl = oracle.attention(pr, f64[0], f64[1][:, :, lo:hi], f64[2][:, :, lo:hi])
        assert_bf16_close(o_r.cpu().numpy().astype(np.float64), ro, f"CP partial W={W} r={r}")
        assert_lse_close(l_r.cpu().numpy(), rl, LSE_TOL_BF16, f"CP partial lse W={W} r={r}")
        o_all[r].copy_(o_r)
        lse_all[r].copy_(l_r)
    out, lse = pdist.merge_prefill_parts(o_all, lse_all, torch.bfloat16)
    assert_bf16_close(out.float().cpu().numpy().astype(np.float64), ref_o, f"CP prefill W={W}")
    assert_lse_close(lse.cpu().numpy(), ref_l, LSE_TOL_BF16, "CP lse")


def test_merge_partials_matches_oracle():
    """attn_merge_partials on oracle-made normalised partials, incl. empty (-inf) parts."""
    P, R, D = 5, 37, 64
    rng = np.random.default_rng(5)
    m = rng.standard_normal((P, R)) * 2
    l = rng.uniform(0.5, 20, (P, R))
    o = rng.standard_normal((P, R, D)) * l[..., None]
    m[1, :10] = -np.inf
    l[1, :10] = 0
    o[1, :10] = 0
    ref_o, ref_l = oracle.splitk_combine(m, l, o)
    live = np.isfinite(m)
    lse_p = np.where(live, m + np.log(np.where(live, l, 1.0)), -np.inf)
    o_norm = np.where(live[..., None], o / np.where(live, l, 1.0)[..., None], 0.0)
    out, lse = pb.merge_partials(torch.tensor(o_norm, dtype=torch.float32, device="cuda"),
                                 torch.tensor(lse_p, dtype=torch.float32, device="cuda"), return_lse=True)
    np.testing.assert_allclose(out.cpu().numpy(), ref_o, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(lse.cpu().numpy(), ref_l, rtol=1e-5, atol=1e-5)


def test_kv_sharded_prefill_nccl_one_rank():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(29900 + os.getpid() % 90))
    created = False
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        created = True
    try:
        B, Hq, Hkv, S, D = 1, 2, 2, 300, 64
        p = problem(B, Hq, Hkv, S, S, D, causal=True)
        raw, f64 = gen_qkv(88, B, Hq, Hkv, S, S, D)
        ref_o, _ = oracle.attention(p, *f64)
        q, k, v = (dgd.to_device(x) for x in raw)
        out, _ = pdist.prefill_kv_sharded(q, k, v, kv_pos_offset=0, seqlen_kv_total=S, causal=True)
        assert_bf16_close(out.float().cpu().numpy().astype(np.float64), ref_o, "CP nccl 1 rank")
    finally:
        if created:
            dist.destroy_process_group()
