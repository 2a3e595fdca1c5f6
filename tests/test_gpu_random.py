"""Randomised GPU parity: seeded random shapes, head layouts, positions, masks, score_mods and
dtypes through the C ABI, element-wise against the fp64 oracle at north_star tolerance.  The
fixed cases elsewhere pin each kernel path; these sweep the corners between them (ragged
Sq / Skv against 64- and 128-key tiles, KV shards, rectangular bottom-right alignment, empty
rows, every GQA group size, both head dims, bf16 and fp16) with one random case per seed."""
import numpy as np
import pytest
import torch

import datagen
import oracle
from datagen import device as dgd
from tests.helpers import LSE_TOL_BF16, assert_bf16_close, assert_lse_close, gen_qkv, problem

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2510_08726_b200 as pb


def _np(t):
    return t.float().cpu().numpy().astype(np.float64)


def _kw(p, hq):
    kw = dict(scale=p.scale, causal=p.causal, window=(p.window_left, p.window_right), softcap=p.softcap,
              kv_pos_offset=p.kv_pos_offset)
    if p.alibi_slopes is not None:
        kw["alibi_slopes"] = torch.tensor(np.asarray(p.alibi_slopes, dtype=np.float32), device="cuda")
    if p.seqlen_kv_total is not None:
        kw["seqlen_kv_total"] = p.seqlen_kv_total
    if p.q_pos_offset is not None:
        kw["q_pos_offset"] = p.q_pos_offset
    return kw


def _random_case(seed, decode=False):
    rng = np.random.default_rng(seed)
    D = int(rng.choice([64, 128]))
    Hkv = int(rng.choice([1, 2, 4]))
    G = int(rng.choice([1, 2, 4] if decode else [1, 2, 4, 8]))
    Hq = Hkv * G
    B = int(rng.integers(1, 3))
    Sq = 1 if decode else int(rng.integers(1, 420))
    Skv = int(rng.integers(1, 900))
    dtype = str(rng.choice(["bf16", "f16"]))
    var = {}
    if rng.random() < 0.5:
        var["causal"] = True
    if rng.random() < 0.3:
        var["window_left"] = int(rng.integers(0, 400))
        if rng.random() < 0.5:
            var["window_right"] = int(rng.integers(0, 100))
    r = rng.random()
    if r < 0.25:
        var["alibi_slopes"] = datagen.alibi_slopes(Hq)
    elif r < 0.45:
        var["softcap"] = float(rng.choice([2.0, 8.0, 50.0]))
    if rng.random() < 0.3:   # a KV shard of a longer sequence (absolute positions)
        total = Skv + int(rng.integers(0, 600))
        var["kv_pos_offset"] = int(rng.integers(0, total - Skv + 1))
        var["seqlen_kv_total"] = total
    if not decode and rng.random() < 0.2:
        var["q_pos_offset"] = int(rng.integers(-50, 1000))
    return B, Hq, Hkv, Sq, Skv, D, dtype, var


@pytest.mark.parametrize("seed", range(120))
def test_random_prefill(seed):
    B, Hq, Hkv, Sq, Skv, D, dtype, var = _random_case(seed)
    p = problem(B, Hq, Hkv, Sq, Skv, D, **var)
    raw, f64 = gen_qkv(20000 + seed, B, Hq, Hkv, Sq, Skv, D, dtype)
    ref_o, ref_l = oracle.attention(p, *f64)
    q, k, v = (dgd.to_device(x, dtype=dtype) for x in raw)
    for splits in (1, 0):   # plain and the library's own KV-split choice
        o, lse = pb.fused_fwd(q, k, v, return_lse=True, kv_splits=splits, **_kw(p, Hq))
        what = f"seed {seed}: B={B} Hq={Hq} Hkv={Hkv} Sq={Sq} Skv={Skv} D={D} {dtype} {var} splits={splits}"
        assert_bf16_close(_np(o), ref_o, what)
        assert_lse_close(lse.cpu().numpy(), ref_l, LSE_TOL_BF16, what + " lse")


@pytest.mark.parametrize("seed", range(64))
def test_random_decode(seed):
    B, Hq, Hkv, Sq, Skv, D, dtype, var = _random_case(1000 + seed, decode=True)
    p = problem(B, Hq, Hkv, Sq, Skv, D, **var)
    raw, f64 = gen_qkv(21000 + seed, B, Hq, Hkv, Sq, Skv, D, dtype)
    ref_o, ref_l = oracle.attention(p, *f64)
    q, k, v = (dgd.to_device(x, dtype=dtype) for x in raw)
    rng = np.random.default_rng(seed)
    splits = int(rng.choice([0, 1, 3, 7]))
    o, lse = pb.splitkv_decode(q, k, v, num_splits=splits, return_lse=True, **_kw(p, Hq))
    what = f"seed {seed}: B={B} Hq={Hq} Hkv={Hkv} Skv={Skv} D={D} {dtype} {var} splits={splits}"
    assert_bf16_close(_np(o), ref_o, what)
    assert_lse_close(lse.cpu().numpy(), ref_l[:, :, 0], LSE_TOL_BF16, what + " lse")
