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


@pytest.mark.parametrize("W", [2, 3, 8])
def test_kv_sharded_decode_loopback(W):
    B, Hq, Hkv, L, D = 2, 8, 2, 3001, 128
    p = problem(B, Hq, Hkv, 1, L, D, causal=True)
    raw, f64 = gen_qkv(900 + W, B, Hq, Hkv, 1, L, D)
    ref_o, ref_l = oracle.attention(p, *f64)
    q, k, v = (dgd.to_device(x) for x in raw)
    packed = torch.empty(W, B, Hq, D + 2, device="cuda")
    for r in range(W):
        lo, hi = pdist.shard_range(L, r, W)
        parts = pdist._local_kernels(q, k[:, :, lo:hi].contiguous(), v[:, :, lo:hi].contiguous(), kv_pos_offset=lo,
                                     seqlen_kv_total=L, num_splits=0, variant=dict(causal=True))
        pdist._merge_kernels(parts, pb.Parts.packed(packed[r:r + 1]))
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
