"""Pins for the fp64 oracle (``oracle/``) against things other than itself:
hand-derived values (tests/golden, each cited), closed forms, invariants, an
independent library (torch CPU fp64 SDPA) and a pure-Python brute force.

Each pin is chosen so a plausible oracle mistake fails it: a dropped scale
(H1, torch), wrong mask direction (H2, H5, H7), wrong ALiBi sign (H3),
missing softcap (H4), wrong GQA mapping (test_gqa_contiguous_groups),
transposed q/k or k/v (torch cross-check with non-square D vs Skv), wrong
empty-row handling (H7)."""
import math

import numpy as np
import pytest
import torch

import datagen
import oracle
from oracle import Problem

INF = float("inf")


def _p_from_case(case, Sq, Skv, D):
    slopes = case.get("alibi_slopes")
    return Problem(batch=1, heads_q=1, heads_kv=1, seqlen_q=Sq, seqlen_kv=Skv, head_dim=D,
                   scale=case["scale"], causal=case.get("causal", False),
                   softcap=case.get("softcap", 0.0),
                   alibi_slopes=None if slopes is None else np.array(slopes),
                   window_left=case.get("window_left", -1), window_right=case.get("window_right", -1))


def _lse(vals):
    return np.array([-INF if v == "-inf" else v for v in vals], dtype=np.float64)


@pytest.mark.parametrize("name", ["H1_softmax_pv", "H2_causal", "H3_alibi_causal", "H4_softcap",
                                  "H5_window", "H7_fully_masked_rows", "H8_splitk_by_hand"])
def test_hand_cases(golden, name):
    c = golden[name]
    q, k, v = (np.array(c[t], dtype=np.float64) for t in ("q", "k", "v"))
    p = _p_from_case(c, q.shape[0], k.shape[0], q.shape[1])
    o, lse = oracle.attention_bh(p, q, k, v, 0)
    np.testing.assert_allclose(o, np.array(c["o"]), rtol=0, atol=1e-15)
    np.testing.assert_allclose(lse, _lse(c["lse"]), rtol=0, atol=1e-15)


def test_hand_splitk_partials(golden):
    c = golden["H8_splitk_by_hand"]
    q, k, v = (np.array(c[t], dtype=np.float64) for t in ("q", "k", "v"))
    p = _p_from_case(c, 1, 4, 1)
    m, l, o = oracle.splitk_local_bh(p, q, k, v, 0, c["split_bounds"])
    np.testing.assert_allclose(m[:, 0], c["part_m"], atol=1e-15)
    np.testing.assert_allclose(l[:, 0], c["part_l"], atol=1e-15)
    np.testing.assert_allclose(o[:, 0, 0], c["part_o"], atol=1e-15)
    out, lse = oracle.splitk_combine(m, l, o)
    np.testing.assert_allclose(out[0], c["o"][0], atol=1e-15)
    np.testing.assert_allclose(lse[0], c["lse"][0], atol=1e-14)


def _rand(shape, seed):
    return np.random.default_rng(seed).standard_normal(shape)


def _torch_ref(p: Problem, q, k, v):
    """Independent library path: torch CPU fp64 SDPA with an additive bias/mask."""
    B, Hq, Sq, D = q.shape
    Skv = k.shape[2]
    qpos = p.q_offset + np.arange(Sq)[:, None]
    kpos = p.kv_pos_offset + np.arange(Skv)[None, :]
    bias = np.zeros((Hq, Sq, Skv))
    if p.alibi_slopes is not None:
        bias -= np.asarray(p.alibi_slopes, dtype=np.float64)[:, None, None] * np.abs(qpos - kpos)[None]
    allowed = np.ones((Sq, Skv), dtype=bool)
    if p.causal:
        allowed &= kpos <= qpos
    if p.window_left >= 0:
        allowed &= qpos - kpos <= p.window_left
    if p.window_right >= 0:
        allowed &= kpos - qpos <= p.window_right
    bias = np.where(allowed[None], bias, -INF)
    G = Hq // k.shape[1]
    kt = torch.from_numpy(k).repeat_interleave(G, dim=1)
    vt = torch.from_numpy(v).repeat_interleave(G, dim=1)
    out = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(q), kt, vt, attn_mask=torch.from_numpy(bias)[None], scale=p.scale)
    return out.numpy()


@pytest.mark.parametrize("variant", ["global", "causal", "window", "alibi", "gqa", "gqa_window_alibi",
                                     "rect_causal", "kv_offset"])
def test_torch_cross_check(variant):
    B, Hq, Hkv, Sq, Skv, D = 2, 4, 4, 37, 53, 24
    kw = {}
    if variant == "causal":
        kw = dict(causal=True)
    elif variant == "window":
        kw = dict(causal=True, window_left=7, window_right=0)
    elif variant == "alibi":
        kw = dict(causal=True, alibi_slopes=datagen.alibi_slopes(Hq))
    elif variant == "gqa":
        Hkv = 2
        kw = dict(causal=True)
    elif variant == "gqa_window_alibi":
        Hkv = 1
        kw = dict(window_left=5, window_right=3, alibi_slopes=datagen.alibi_slopes(Hq))
    elif variant == "rect_causal":
        Sq = 20
        kw = dict(causal=True)
    elif variant == "kv_offset":
        # KV shard [10, 63) of a 63-long sequence; queries at the end: bottom-right causal
        kw = dict(causal=True, seqlen_kv_total=Skv + 10, kv_pos_offset=10, q_pos_offset=Skv + 10 - Sq)
    p = Problem(B, Hq, Hkv, Sq, Skv, D, scale=1 / math.sqrt(D), **kw)
    q, k, v = _rand((B, Hq, Sq, D), 1), _rand((B, Hkv, Skv, D), 2), _rand((B, Hkv, Skv, D), 3)
    o, lse = oracle.attention(p, q, k, v)
    ref = _torch_ref(p, q, k, v)
    live = np.isfinite(lse)
    assert live.all(), "choose shapes without fully masked rows for the torch check"
    np.testing.assert_allclose(o, ref, rtol=0, atol=1e-12)


def _brute(p: Problem, q, k, v, hq):
    """Pure-Python brute force (math module, fsum), one row at a time."""
    Sq, D = q.shape
    out, lses = [], []
    for i in range(Sq):
        qpos = p.q_offset + i
        xs, vs = [], []
        for j in range(k.shape[0]):
            kpos = p.kv_pos_offset + j
            if p.causal and kpos > qpos:
                continue
            if p.window_left >= 0 and qpos - kpos > p.window_left:
                continue
            if p.window_right >= 0 and kpos - qpos > p.window_right:
                continue
            x = p.scale * math.fsum(q[i, d] * k[j, d] for d in range(D))
            if p.softcap > 0:
                x = p.softcap * math.tanh(x / p.softcap)
            if p.alibi_slopes is not None:
                x -= float(p.alibi_slopes[hq]) * abs(qpos - kpos)
            xs.append(x)
            vs.append(v[j])
        if not xs:
            out.append([0.0] * v.shape[1])
            lses.append(-INF)
            continue
        m = max(xs)
        w = [math.exp(x - m) for x in xs]
        l = math.fsum(w)
        out.append([math.fsum(wi * vj[d] for wi, vj in zip(w, vs)) / l for d in range(v.shape[1])])
        lses.append(m + math.log(l))
    return np.array(out), np.array(lses)


@pytest.mark.parametrize("kw", [dict(), dict(causal=True), dict(softcap=2.0, causal=True),
                                dict(window_left=3, window_right=2, alibi=True),
                                dict(causal=True, Sq=9, Skv=4)])
def test_brute_force_tiny(kw):
    kw = dict(kw)
    Sq, Skv = kw.pop("Sq", 7), kw.pop("Skv", 11)
    alibi = kw.pop("alibi", False)
    D = 5
    p = Problem(1, 2, 1, Sq, Skv, D, scale=0.7, alibi_slopes=datagen.alibi_slopes(2) if alibi else None, **kw)
    q, k, v = _rand((2, Sq, D), 4), _rand((Skv, D), 5), _rand((Skv, D), 6)
    for hq in range(2):
        o, lse = oracle.attention_bh(p, q[hq], k, v, hq)
        ob, lb = _brute(p, q[hq], k, v, hq)
        np.testing.assert_allclose(o, ob, rtol=0, atol=1e-13)
        np.testing.assert_allclose(lse, lb, rtol=0, atol=1e-13)


def test_softcap_closed_form_large_cap_is_identity():
    """I5: cap -> infinity reduces softcap to plain attention."""
    p0 = Problem(1, 1, 1, 16, 16, 8, scale=0.3)
    p1 = Problem(1, 1, 1, 16, 16, 8, scale=0.3, softcap=1e7)
    q, k, v = _rand((16, 8), 7), _rand((16, 8), 8), _rand((16, 8), 9)
    np.testing.assert_allclose(oracle.attention_bh(p1, q, k, v, 0)[0], oracle.attention_bh(p0, q, k, v, 0)[0], atol=1e-10)


def test_softcap_changes_result():
    """cap = 2 must visibly differ from no softcap (a dropped softcap fails here)."""
    p0 = Problem(1, 1, 1, 16, 16, 8, scale=1.0)
    p1 = Problem(1, 1, 1, 16, 16, 8, scale=1.0, softcap=2.0)
    q, k, v = _rand((16, 8), 7), _rand((16, 8), 8), _rand((16, 8), 9)
    assert np.abs(oracle.attention_bh(p1, q, k, v, 0)[0] - oracle.attention_bh(p0, q, k, v, 0)[0]).max() > 1e-2


def test_rows_sum_to_one_via_identity_v():
    """I1: with V = I (Dv = Skv) the output row IS the softmax row: sums to 1."""
    Skv = 19
    p = Problem(1, 1, 1, 13, Skv, 6, scale=0.5, causal=True, alibi_slopes=np.array([0.25]))
    q, k = _rand((13, 6), 10), _rand((Skv, 6), 11)
    o, lse = oracle.attention_bh(p, q, k, np.eye(Skv), 0)
    np.testing.assert_allclose(o.sum(axis=1), 1.0, atol=1e-12)
    assert (o >= 0).all()


def test_constant_v_and_zero_q():
    """I2: V = c => O = c. I3: Q = 0 without bias => O = mean of allowed V rows (causal prefix mean)."""
    p = Problem(1, 1, 1, 12, 12, 4, scale=1.0, causal=True)
    q, k = _rand((12, 4), 12), _rand((12, 4), 13)
    o, _ = oracle.attention_bh(p, q, k, np.full((12, 3), 2.5), 0)
    np.testing.assert_allclose(o, 2.5, atol=1e-13)
    v = _rand((12, 3), 14)
    o, _ = oracle.attention_bh(p, np.zeros((12, 4)), k, v, 0)
    prefix = np.cumsum(v, axis=0) / np.arange(1, 13)[:, None]
    np.testing.assert_allclose(o, prefix, atol=1e-13)


def test_kv_permutation_invariance():
    """I4: jointly permuting K, V rows leaves non-causal, bias-free output unchanged."""
    p = Problem(1, 1, 1, 9, 15, 4, scale=0.8)
    q, k, v = _rand((9, 4), 15), _rand((15, 4), 16), _rand((15, 4), 17)
    perm = np.random.default_rng(0).permutation(15)
    np.testing.assert_allclose(oracle.attention_bh(p, q, k[perm], v[perm], 0)[0],
                               oracle.attention_bh(p, q, k, v, 0)[0], atol=1e-13)


def test_window_covering_everything_equals_causal():
    """I5: window >= Skv reduces to causal."""
    p0 = Problem(1, 1, 1, 20, 20, 4, scale=0.8, causal=True)
    p1 = Problem(1, 1, 1, 20, 20, 4, scale=0.8, window_left=100, window_right=0)
    q, k, v = _rand((20, 4), 18), _rand((20, 4), 19), _rand((20, 4), 20)
    np.testing.assert_allclose(oracle.attention_bh(p1, q, k, v, 0)[0], oracle.attention_bh(p0, q, k, v, 0)[0], atol=1e-14)


def test_single_token_returns_v():
    """I6: S_q = S_kv = 1 => O = v."""
    p = Problem(1, 1, 1, 1, 1, 3, scale=1.0, causal=True)
    v = np.array([[1.5, -2.0, 0.25]])
    o, _ = oracle.attention_bh(p, _rand((1, 3), 21), _rand((1, 3), 22), v, 0)
    np.testing.assert_array_equal(o, v)


def test_gqa_contiguous_groups():
    """R6 reading: q-head hq uses kv-head hq // G (contiguous groups), not hq % Hkv."""
    B, Hq, Hkv, S, D = 1, 4, 2, 6, 3
    p = Problem(B, Hq, Hkv, S, S, D, scale=1.0)
    q = _rand((B, Hq, S, D), 23)
    k, v = _rand((B, Hkv, S, D), 24), _rand((B, Hkv, S, D), 25)
    o, _ = oracle.attention(p, q, k, v)
    ph = Problem(1, 1, 1, S, S, D, scale=1.0)
    for hq, g in [(0, 0), (1, 0), (2, 1), (3, 1)]:
        np.testing.assert_allclose(o[0, hq], oracle.attention_bh(ph, q[0, hq], k[0, g], v[0, g], 0)[0], atol=1e-14)
    # heads 1 and 2 differ in group under this reading
    assert oracle.head_group(p, 1) == 0 and oracle.head_group(p, 2) == 1
