"""World-size-2 gloo test of the KV-sharded decode plumbing (dist.py) on CPU:
shard ranges and position offsets, the packed [B, H, D+2] all-gather layout,
and the two-level merge.  The local section / merges are injected with
oracle-backed stand-ins (the CUDA kernels are covered by test_gpu_parity)."""
import math
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen
import oracle
from paper_2510_08726_b200 import Parts
from paper_2510_08726_b200 import dist as pdist

B, Hq, Hkv, L, D = 2, 4, 2, 203, 16


def _problem(**kw):
    return oracle.Problem(B, Hq, Hkv, 1, L, D, scale=1 / math.sqrt(D), causal=True, **kw)


def _inputs():
    q = datagen.as_f64(datagen.tensor(11, 1, (B, Hq, 1, D)), "bf16")
    k = datagen.as_f64(datagen.tensor(11, 2, (B, Hkv, L, D)), "bf16")
    v = datagen.as_f64(datagen.tensor(11, 3, (B, Hkv, L, D)), "bf16")
    return q, k, v


def _local(q, k_shard, v_shard, *, kv_pos_offset, seqlen_kv_total, num_splits, variant):
    """Stand-in for the decode kernel: oracle Split-K local section over this shard."""
    Ls = k_shard.shape[2]
    p = oracle.Problem(B, Hq, Hkv, 1, Ls, D, scale=1 / math.sqrt(D), causal=True, kv_pos_offset=kv_pos_offset,
                       seqlen_kv_total=seqlen_kv_total)
    bounds = [0, Ls // 3, Ls]
    m = np.zeros((2, B, Hq)); l = np.zeros((2, B, Hq)); o = np.zeros((2, B, Hq, D))
    for b in range(B):
        for hq in range(Hq):
            g = oracle.head_group(p, hq)
            mm, ll, oo = oracle.splitk_local_bh(p, q[b, hq].numpy(), k_shard[b, g].numpy(), v_shard[b, g].numpy(),
                                                hq, bounds)
            m[:, b, hq], l[:, b, hq], o[:, b, hq] = mm[:, 0], ll[:, 0], oo[:, 0]
    t = lambda x: torch.tensor(x, dtype=torch.float32)  # noqa: E731
    return Parts(t(m), t(l), t(o))


def _merge(parts, acc):
    M, Lm, O = oracle.splitk_merge(parts.m.double().numpy(), parts.l.double().numpy(), parts.o.double().numpy())
    acc.m.copy_(torch.tensor(M)[None]); acc.l.copy_(torch.tensor(Lm)[None]); acc.o.copy_(torch.tensor(O)[None])


def _final(parts, dtype, return_lse):
    out, lse = oracle.splitk_combine(parts.m.double().numpy(), parts.l.double().numpy(), parts.o.double().numpy())
    return torch.tensor(out)[:, :, None], torch.tensor(lse)


def _worker(rank, world, port, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q, k, v = _inputs()
    lo, hi = pdist.shard_range(L, rank, world)
    out, lse = pdist.decode_kv_sharded(torch.tensor(q), torch.tensor(k[:, :, lo:hi]), torch.tensor(v[:, :, lo:hi]),
                                       kv_pos_offset=lo, seqlen_kv_total=L, local=_local, merge=_merge,
                                       final=_final, return_lse=True)
    np.save(os.path.join(result_dir, f"out{rank}.npy"), out.numpy())
    np.save(os.path.join(result_dir, f"lse{rank}.npy"), lse.numpy())
    dist.destroy_process_group()


def test_shard_range_covers_everything():
    for n in (1, 7, 203, 131072):
        for w in (1, 2, 3, 8):
            spans = [pdist.shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_kv_sharded_decode_two_ranks(tmp_path):
    port = 29500 + os.getpid() % 1000
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    q, k, v = _inputs()
    ref_o, ref_l = oracle.attention(_problem(), q, k, v)
    for r in range(2):
        out = np.load(tmp_path / f"out{r}.npy")
        lse = np.load(tmp_path / f"lse{r}.npy")
        np.testing.assert_allclose(out, ref_o, atol=2e-6)       # fp32 gather of fp64 partials
        np.testing.assert_allclose(lse, ref_l[:, :, 0], atol=2e-6)


def _prefill_local_oracle(q, k_shard, v_shard, *, kv_pos_offset, seqlen_kv_total, variant):
    """Stand-in for the Rolling Update kernel on one KV shard: oracle O and lse."""
    Bq, Hq_, S, Dd = q.shape
    p = oracle.Problem(Bq, Hq_, k_shard.shape[1], S, k_shard.shape[2], Dd, scale=1 / math.sqrt(Dd), causal=True,
                       kv_pos_offset=kv_pos_offset, seqlen_kv_total=seqlen_kv_total)
    o, lse = oracle.attention(p, q.numpy(), k_shard.numpy(), v_shard.numpy())
    return torch.tensor(o), torch.tensor(lse)


def _prefill_final_oracle(o_all, lse_all, out_dtype):
    o, l = o_all.numpy(), lse_all.numpy()
    live = np.isfinite(l)
    out, lse = oracle.splitk_combine(np.where(live, l, -np.inf), live.astype(float), o)
    return torch.tensor(out), torch.tensor(lse)


def _cp_worker(rank, world, port, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    S = 57
    q = datagen.as_f64(datagen.tensor(12, 1, (1, 2, S, 8)), "bf16")
    k = datagen.as_f64(datagen.tensor(12, 2, (1, 2, S, 8)), "bf16")
    v = datagen.as_f64(datagen.tensor(12, 3, (1, 2, S, 8)), "bf16")
    lo, hi = pdist.shard_range(S, rank, world)
    out, lse = pdist.prefill_kv_sharded(torch.tensor(q), torch.tensor(k[:, :, lo:hi]), torch.tensor(v[:, :, lo:hi]),
                                        kv_pos_offset=lo, seqlen_kv_total=S, local=_prefill_local_oracle,
                                        final=_prefill_final_oracle)
    np.save(os.path.join(result_dir, f"cp{rank}.npy"), out.numpy())
    dist.destroy_process_group()


def test_kv_sharded_prefill_two_ranks(tmp_path):
    port = 29400 + os.getpid() % 100
    mp.spawn(_cp_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    S = 57
    q = datagen.as_f64(datagen.tensor(12, 1, (1, 2, S, 8)), "bf16")
    k = datagen.as_f64(datagen.tensor(12, 2, (1, 2, S, 8)), "bf16")
    v = datagen.as_f64(datagen.tensor(12, 3, (1, 2, S, 8)), "bf16")
    ref, _ = oracle.attention(oracle.Problem(1, 2, 2, S, S, 8, scale=1 / math.sqrt(8), causal=True), q, k, v)
    for r in range(2):
        np.testing.assert_allclose(np.load(tmp_path / f"cp{r}.npy"), ref, atol=1e-12)
