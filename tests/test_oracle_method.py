"""The paper's repaired fusions (Rolling Update, Split-K Update, Fig. 2 chain)
written step by step in ``oracle/`` must equal the unfused definition for ANY
tile / split / shard partition (Thms. 1-4; Eq. 8), and
naive fusion without repair must NOT (Fig. 2b)."""
import math

import numpy as np
import pytest

import datagen
import oracle
from oracle import Problem


def _rand(shape, seed):
    return np.random.default_rng(seed).standard_normal(shape)


def _random_bounds(n, rng, max_parts=9, allow_empty=False):
    k = int(rng.integers(1, max_parts + 1))
    cuts = np.sort(rng.integers(0 if allow_empty else 1, n + (1 if allow_empty else 0), size=k - 1))
    b = [0] + [int(c) for c in cuts] + [n]
    if not allow_empty:
        b = sorted(set(b))
    return b


VARIANTS = [dict(), dict(causal=True), dict(causal=True, alibi=True), dict(causal=True, softcap=2.0),
            dict(window_left=9, window_right=0), dict(window_left=4, window_right=6, alibi=True)]


def _prob(kw, Sq=23, Skv=41, D=8, Hq=2):
    kw = dict(kw)
    alibi = kw.pop("alibi", False)
    return Problem(1, Hq, 1, Sq, Skv, D, scale=1 / math.sqrt(D),
                   alibi_slopes=datagen.alibi_slopes(Hq) if alibi else None, **kw)


@pytest.mark.parametrize("vi", range(len(VARIANTS)))
def test_R1_rolling_update_equals_definition(vi):
    """R1: Fig. 19 rolling update over random non-uniform tiles (incl. size 1 and a single tile)."""
    p = _prob(VARIANTS[vi])
    q, k, v = _rand((23, 8), 1), _rand((41, 8), 2), _rand((41, 8), 3) * 3
    ref_o, ref_l = oracle.attention_bh(p, q, k, v, 1)
    rng = np.random.default_rng(vi)
    tilings = [[0, 41], list(range(42))] + [_random_bounds(41, rng) for _ in range(20)]
    for b in tilings:
        o, l = oracle.rolling_update_bh(p, q, k, v, 1, b)
        np.testing.assert_allclose(o, ref_o, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(l, ref_l, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("vi", range(len(VARIANTS)))
def test_R2_splitk_equals_definition(vi):
    """R2: Fig. 5 / Eq. 8 with random partition counts, incl. empty and fully masked parts."""
    p = _prob(VARIANTS[vi])
    q, k, v = _rand((23, 8), 4), _rand((41, 8), 5), _rand((41, 8), 6)
    ref_o, ref_l = oracle.attention_bh(p, q, k, v, 0)
    rng = np.random.default_rng(100 + vi)
    for _ in range(20):
        b = _random_bounds(41, rng, max_parts=12, allow_empty=True)
        m, l, o = oracle.splitk_local_bh(p, q, k, v, 0, b)
        out, lse = oracle.splitk_combine(m, l, o)
        np.testing.assert_allclose(out, ref_o, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(lse, ref_l, rtol=1e-12, atol=1e-12)


def test_R3_hierarchical_combine_is_associative():
    """R3: splits within shards, then shards, in arbitrary grouping and order (Eq. 4)."""
    p = _prob(dict(causal=True, alibi=True), Sq=5, Skv=64)
    q, k, v = _rand((5, 8), 7), _rand((64, 8), 8), _rand((64, 8), 9)
    ref_o, ref_l = oracle.attention_bh(p, q, k, v, 0)
    b = [0, 3, 10, 10, 17, 30, 41, 50, 64]
    m, l, o = oracle.splitk_local_bh(p, q, k, v, 0, b)
    rng = np.random.default_rng(3)
    for _ in range(10):
        perm = rng.permutation(len(m))
        groups = np.array_split(perm, int(rng.integers(1, 5)))
        tri = [oracle.splitk_merge(m[g], l[g], o[g]) for g in groups if len(g)]
        M = np.stack([t[0] for t in tri]); L = np.stack([t[1] for t in tri]); O = np.stack([t[2] for t in tri])
        out, lse = oracle.splitk_combine(M, L, O)
        np.testing.assert_allclose(out, ref_o, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(lse, ref_l, rtol=1e-12, atol=1e-12)


def test_R4_naive_fusion_without_repair_is_wrong(golden):
    """R4 negative control (Fig. 2b): dropping the repair term breaks the result,
    so the R1/R2 tests can detect a missing repair."""
    rng = np.random.default_rng(4)
    inp = rng.standard_normal((8, 64))
    ref = oracle.softmax_denominator(inp)
    assert np.abs(oracle.softmax_denominator_naive_fused(inp) - ref).max() > 1e-3
    np.testing.assert_allclose(oracle.softmax_denominator_rolling(inp), ref, rtol=1e-12)
    c = golden["FIG2_softmax_denominator"]
    inp = np.array(c["inp"])
    np.testing.assert_allclose(oracle.softmax_denominator(inp), c["xsum"], atol=1e-15)
    np.testing.assert_allclose(oracle.softmax_denominator_rolling(inp), c["xsum"], atol=1e-15)


def test_fig2_trace_example_result(golden):
    """Eq. example-result: the repaired s<3> equals the original s<3> while
    s<j>, j < 3, differs from the original program's partial sums."""
    c = golden["FIG2_softmax_denominator"]
    inp = np.array(c["inp"])
    xsum, hist = oracle.softmax_denominator_rolling(inp, trace=True)
    np.testing.assert_allclose(hist[0], c["trace_row0"], atol=1e-15)
    orig_partial = np.cumsum(np.exp(inp[0] - inp[0].max()))
    assert np.all(np.abs(hist[0, :3] - orig_partial[:3]) > 1e-3)
    assert abs(hist[0, 3] - orig_partial[3]) < 1e-15
    # row 1 has its max first: the repair term is always 1 and the traces coincide
    np.testing.assert_allclose(hist[1], np.cumsum(np.exp(inp[1] - 3.0)), atol=1e-15)


def test_fig19_and_fig5_softmax_chain():
    rng = np.random.default_rng(5)
    for _ in range(100):
        inp = rng.standard_normal((2, 8)) * 4
        ref = oracle.softmax_denominator(inp)
        np.testing.assert_allclose(oracle.softmax_denominator_privatized(inp, 2), ref, rtol=1e-12)
        mg, sg = oracle.softmax_denominator_splitk(inp, 4)
        np.testing.assert_allclose(sg, ref, rtol=1e-12)
        np.testing.assert_array_equal(mg, inp.max(axis=1))


def test_R5_R6_R7_repair_algebra():
    """R5 Def. 1 tag-update, R6 Thm. 2 round trip g(x, g_c^-1(x, y)) = y for
    g(x, c) = exp(c - x), R7 Eq. 4 h(x + y) = h(x) + h(y); >= 1000 cases."""
    rng = np.random.default_rng(6)
    n = 2000
    x, r, r2 = rng.standard_normal(n) * 3, rng.standard_normal(n) * 3, rng.standard_normal(n) * 3
    y = np.exp(rng.standard_normal(n))
    # R6: g_c^-1(x, y) = x + ln y  (Fig. 18d)
    np.testing.assert_allclose(np.exp((x + np.log(y)) - x), y, rtol=1e-12)
    # Eq. 5 condition 1: h(g(r, c), r, r') = g(r', c)
    c = rng.standard_normal(n)
    np.testing.assert_allclose(oracle.repair_h(np.exp(c - r), r, r2), np.exp(c - r2), rtol=1e-12)
    # R7: h distributes over f = +
    a, b = rng.standard_normal(n), rng.standard_normal(n)
    np.testing.assert_allclose(oracle.repair_h(a + b, r, r2), oracle.repair_h(a, r, r2) + oracle.repair_h(b, r, r2),
                               rtol=1e-12, atol=1e-12)
    # R5: h tag-updates a whole reduce expression sum_{j'<=j} g(X_r<j>, c_j') to X_r<j+1>
    for t in range(200):
        cs = rng.standard_normal(8)
        m_j, m_next = rng.standard_normal(2)
        lhs = oracle.repair_h(np.sum(np.exp(cs - m_j)), m_j, m_next)
        np.testing.assert_allclose(lhs, np.sum(np.exp(cs - m_next)), rtol=1e-12)


@pytest.mark.parametrize("tau", [0.0, 1.0, 5.545177444479562, 50.0])
def test_R8_lazy_rescale_equals_definition(tau):
    """R8: stale-reference rolling update (any r', Thm. 2) equals the definition; tau = 0 is
    the eager schedule. 5.545 = 8 ln 2, the kernel's threshold (8 in log2 units)."""
    p = _prob(dict(causal=True, alibi=True), Sq=31, Skv=97)
    q, k, v = _rand((31, 8), 10) * 2, _rand((97, 8), 11) * 2, _rand((97, 8), 12)
    ref_o, ref_l = oracle.attention_bh(p, q, k, v, 1)
    rng = np.random.default_rng(7)
    for b in [list(range(0, 98, 16)) + [97], _random_bounds(97, rng), list(range(98))]:
        o, l = oracle.rolling_update_lazy_bh(p, q, k, v, 1, b, tau)
        np.testing.assert_allclose(o, ref_o, rtol=1e-11, atol=1e-12)
        np.testing.assert_allclose(l, ref_l, rtol=1e-12, atol=1e-12)


def test_softmax_rows_pins(golden):
    """oracle.softmax_rows (vectorised Fig. 2a) against the Fig. 2 golden values, the
    loop-for-loop Fig. 2a/2c programs, scipy's logsumexp and softmax invariants."""
    from scipy.special import logsumexp
    c = golden["FIG2_softmax_denominator"]
    m, l, y = oracle.softmax_rows(np.array(c["inp"]))
    np.testing.assert_allclose(l, c["xsum"], atol=1e-15)
    np.testing.assert_array_equal(m, [3.0, 3.0])
    rng = np.random.default_rng(11)
    x = rng.standard_normal((6, 37)) * 5
    x[2, 1::3] = -np.inf
    m, l, y = oracle.softmax_rows(x)
    np.testing.assert_allclose(l, oracle.softmax_denominator(x), rtol=1e-13)
    np.testing.assert_allclose(l, oracle.softmax_denominator_rolling(x), rtol=1e-12)
    np.testing.assert_allclose(m + np.log(l), logsumexp(x, axis=1), rtol=1e-13)
    np.testing.assert_allclose(y.sum(axis=1), 1.0, atol=1e-13)
    np.testing.assert_allclose(oracle.softmax_rows(x + 7.25)[2], y, atol=1e-15)   # shift invariance
    z = np.full((2, 5), -np.inf)
    zm, zl, zy = oracle.softmax_rows(z)
    assert np.all(zm == -np.inf) and np.all(zl == 0) and np.all(zy == 0)
