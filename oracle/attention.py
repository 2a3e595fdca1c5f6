"""Plain fp64 attention as the paper defines it, plus the paper's two repaired
fusions written out step by step (CPU, slow, obviously correct).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

* ``attention`` / ``attention_bh`` -- the DEFINITION: Fig. 8's compute
  definition: ``p = q k^T``, ``score_mod`` / mask
  (P:1379-1383), ``softmax_maxelem``, ``softmax_exp``
  (P:1389-1393), ``softmax_expsum``, ``sv = s_exp v``
  (P:1402), ``softmax_norm``. S is materialised (in row blocks),
  nothing is fused or reordered. GQA (excluded from Fig. 8) uses the
  contiguous-group reading ``hkv = hq // (Hq / Hkv)`` (R6).
* ``rolling_update_bh`` -- Rolling Update (Alg. 1) in its tiled
  form (privatization + rolling update, Fig. 19): per KV tile a
  local max, the global max, the repair term ``h(t, r, r') = exp(r - r') t``
  (Fig. 18d) applied to the running sum and to the PV
  accumulator (Eq. 7), then ``m_old <- m_new`` (Alg. 1
  CacheReducePrevResult).
* ``rolling_update_lazy_bh`` -- the same recurrence, but the reference max is
  only moved when it grows by more than ``tau``. Exact in real arithmetic
  because h tag-updates to ANY reference r' (Thm. 2 / Eq. 6).
  This is the schedule the tcgen05 kernel runs (R9).
* ``splitk_local_bh`` / ``splitk_combine`` / ``splitk_merge`` -- Split-K
  Update (Alg. 2; Fig. 5): independent local sections
  producing (max_l, sum_l, PV_l), then the global section with the repair
  term on the right of the reducer (Eq. 8).

Conventions (binding here and in DESIGN.md):
positions ``qpos(i) = q_pos_offset + i``, ``kpos(j) = kv_pos_offset + j``,
``q_pos_offset`` defaults to ``seqlen_kv_total - seqlen_q`` (bottom-right
causal alignment, R7); order inside score_mod is scale -> softcap -> ALiBi ->
mask (R2); softcap ``x = c tanh(x / c)`` (R3); ALiBi bias
``-slope[hq] |qpos - kpos|`` (R4); a fully masked row gives O = 0 and
lse = -inf (R8); ``exp(-inf) = 0``.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

NEG_INF = -np.inf


@dataclass
class Problem:
    batch: int
    heads_q: int
    heads_kv: int
    seqlen_q: int
    seqlen_kv: int
    head_dim: int
    scale: float
    softcap: float = 0.0
    alibi_slopes: Optional[np.ndarray] = None   # fp32 [heads_q]
    causal: bool = False
    window_left: int = -1
    window_right: int = -1
    seqlen_kv_total: Optional[int] = None
    q_pos_offset: Optional[int] = None
    kv_pos_offset: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def kv_total(self) -> int:
        return self.seqlen_kv if self.seqlen_kv_total is None else self.seqlen_kv_total

    @property
    def q_offset(self) -> int:
        return self.kv_total - self.seqlen_q if self.q_pos_offset is None else self.q_pos_offset


def head_group(p: Problem, hq: int) -> int:
    """GQA mapping (reading R6): contiguous groups of G = Hq / Hkv query heads."""
    return hq // (p.heads_q // p.heads_kv)


def _scores(p: Problem, q_rows: np.ndarray, rows: np.ndarray, k: np.ndarray, hq: int,
            j0: int = 0, j1: Optional[int] = None) -> np.ndarray:
    """score_mod(p) masked to -inf, Fig. 8 lines P:1378-1383, for query rows
    ``rows`` against keys j0..j1 of ``k``. Returns fp64 [len(rows), j1 - j0]."""
    j1 = k.shape[0] if j1 is None else j1
    x = p.scale * (q_rows @ k[j0:j1].T)                                   # P:1378, R1
    if p.softcap > 0.0:                                                   # R3
        x = p.softcap * np.tanh(x / p.softcap)
    qpos = (p.q_offset + rows.astype(np.int64))[:, None]
    kpos = (p.kv_pos_offset + np.arange(j0, j1, dtype=np.int64))[None, :]
    if p.alibi_slopes is not None:                                        # R4
        slope = float(p.alibi_slopes[hq])
        x = x - slope * np.abs(qpos - kpos).astype(np.float64)
    allowed = np.ones(x.shape, dtype=bool)
    if p.causal:
        allowed &= kpos <= qpos
    if p.window_left >= 0:
        allowed &= (qpos - kpos) <= p.window_left
    if p.window_right >= 0:
        allowed &= (kpos - qpos) <= p.window_right
    return np.where(allowed, x, NEG_INF)                                  # if_then_else(mask, ., -inf)


def attention_bh(p: Problem, q: np.ndarray, k: np.ndarray, v: np.ndarray, hq: int,
                 rows: Optional[Sequence[int]] = None, row_block: int = 512):
    """Unfused attention for one (b, hq): q [Sq, D], k/v [Skv, D] (fp64).

    Returns (O [R, D], lse [R]) for the requested rows (default: all)."""
    rows = np.arange(q.shape[0]) if rows is None else np.asarray(rows, dtype=np.int64)
    out = np.zeros((len(rows), v.shape[1]))
    lse = np.full(len(rows), NEG_INF)
    for r0 in range(0, len(rows), row_block):
        rr = rows[r0:r0 + row_block]
        s = _scores(p, q[rr], rr, k, hq)                                  # materialise S
        m = s.max(axis=1)                                                 # softmax_maxelem P:1385-1388
        live = m > NEG_INF                                                # R8: fully masked rows
        m_safe = np.where(live, m, 0.0)
        e = np.exp(s - m_safe[:, None])                                   # softmax_exp P:1389-1393
        l = e.sum(axis=1)                                                 # softmax_expsum P:1394-1397
        sv = e @ v                                                        # batch_matmul_NN P:1402
        with np.errstate(invalid="ignore", divide="ignore"):
            o = sv / l[:, None]                                           # softmax_norm P:1403-1406
            lse_b = m + np.log(l)
        out[r0:r0 + len(rr)] = np.where(live[:, None], o, 0.0)
        lse[r0:r0 + len(rr)] = np.where(live, lse_b, NEG_INF)
    return out, lse


def attention(p: Problem, q: np.ndarray, k: np.ndarray, v: np.ndarray):
    """Full unfused attention. q [B, Hq, Sq, D], k/v [B, Hkv, Skv, D] (fp64).
    Returns (O [B, Hq, Sq, D], lse [B, Hq, Sq])."""
    B, Hq, Sq, D = q.shape
    o = np.zeros((B, Hq, Sq, v.shape[-1]))
    lse = np.zeros((B, Hq, Sq))
    for b in range(B):
        for hq in range(Hq):
            g = head_group(p, hq)
            o[b, hq], lse[b, hq] = attention_bh(p, q[b, hq], k[b, g], v[b, g], hq)
    return o, lse


def _tile_bounds(bounds: Sequence[int]):
    return list(zip(bounds[:-1], bounds[1:]))


def rolling_update_bh(p: Problem, q: np.ndarray, k: np.ndarray, v: np.ndarray, hq: int,
                      bounds: Sequence[int], rows: Optional[Sequence[int]] = None):
    """Rolling Update over KV tiles [bounds[t], bounds[t+1]) (Fig. 19 form).

    Per tile: local max (Fig. 19 ``max_local``), global max (``max_global``),
    repair h = exp(m_old - m_new) * t on l and O (Eq. 7, Fig. 18d), local sum
    and local PV, then m_old <- m_new."""
    rows = np.arange(q.shape[0]) if rows is None else np.asarray(rows, dtype=np.int64)
    R, Dv = len(rows), v.shape[1]
    m_old = np.full(R, NEG_INF)              # xmax_0 = -inf (Fig. 2c; SPEC S:304 identity init)
    l = np.zeros(R)
    acc = np.zeros((R, Dv))
    for j0, j1 in _tile_bounds(bounds):
        x = _scores(p, q[rows], rows, k, hq, j0, j1)
        m_loc = x.max(axis=1) if j1 > j0 else np.full(R, NEG_INF)        # xmax_1p
        m_new = np.maximum(m_old, m_loc)                                  # xmax_1
        live = m_new > NEG_INF
        # repair term h(t, r, r') = exp(r - r') t; guard m_new = -inf => alpha = 1 (R8)
        alpha = np.where(live, np.exp(np.where(live, m_old - np.where(live, m_new, 0.0), 0.0)), 1.0)
        e = np.exp(x - np.where(live, m_new, 0.0)[:, None])              # exp(x - xmax_1)
        l = alpha * l + e.sum(axis=1)                                     # xsum = h(xsum) + xsump
        acc = alpha[:, None] * acc + e @ v[j0:j1]                         # O = h(O) + P V_j
        m_old = m_new                                                     # xmax_0 = xmax_1
    live = l > 0
    with np.errstate(invalid="ignore", divide="ignore"):
        out = np.where(live[:, None], acc / l[:, None], 0.0)
        lse = np.where(live, m_old + np.log(l), NEG_INF)
    return out, lse


def rolling_update_lazy_bh(p: Problem, q: np.ndarray, k: np.ndarray, v: np.ndarray, hq: int,
                           bounds: Sequence[int], tau: float, rows: Optional[Sequence[int]] = None):
    """Rolling Update with a stale reference r' (reading R9).

    The reference m_ref moves to the running max only when that max exceeds
    it by more than ``tau``; otherwise p = exp(x - m_ref) <= e^tau. h repairs
    to any reference (Eq. 6), so the final O / l is unchanged."""
    rows = np.arange(q.shape[0]) if rows is None else np.asarray(rows, dtype=np.int64)
    R, Dv = len(rows), v.shape[1]
    m_ref = np.full(R, NEG_INF)
    l = np.zeros(R)
    acc = np.zeros((R, Dv))
    for j0, j1 in _tile_bounds(bounds):
        x = _scores(p, q[rows], rows, k, hq, j0, j1)
        m_loc = x.max(axis=1) if j1 > j0 else np.full(R, NEG_INF)
        m_run = np.maximum(m_ref, m_loc)
        move = (m_run > NEG_INF) & ((m_ref == NEG_INF) | (m_run - m_ref > tau))
        new_ref = np.where(move, m_run, m_ref)
        live = new_ref > NEG_INF
        alpha = np.where(move & (m_ref > NEG_INF), np.exp(m_ref - np.where(live, new_ref, 0.0)), 1.0)
        alpha = np.where(move & (m_ref == NEG_INF), 0.0, alpha)        # first finite reference: O, l are 0
        e = np.exp(x - np.where(live, new_ref, 0.0)[:, None])
        e = np.where(live[:, None], e, 0.0)
        l = alpha * l + e.sum(axis=1)
        acc = alpha[:, None] * acc + e @ v[j0:j1]
        m_ref = new_ref
    live = l > 0
    with np.errstate(invalid="ignore", divide="ignore"):
        out = np.where(live[:, None], acc / l[:, None], 0.0)
        lse = np.where(live, m_ref + np.log(l), NEG_INF)
    return out, lse


def splitk_local_bh(p: Problem, q: np.ndarray, k: np.ndarray, v: np.ndarray, hq: int,
                    bounds: Sequence[int], rows: Optional[Sequence[int]] = None):
    """Split-K local section (Fig. 5 ``s_max_local`` / ``s_sum_local`` plus the
    local PV). For each split s = [bounds[s], bounds[s+1]):
    m_s = max x, l_s = sum exp(x - m_s), O_s = sum exp(x - m_s) v (un-normalised).
    Empty or fully masked split: (-inf, 0, 0). Returns m, l [S, R], O [S, R, D]."""
    rows = np.arange(q.shape[0]) if rows is None else np.asarray(rows, dtype=np.int64)
    spans = _tile_bounds(bounds)
    R, Dv = len(rows), v.shape[1]
    m = np.full((len(spans), R), NEG_INF)
    l = np.zeros((len(spans), R))
    o = np.zeros((len(spans), R, Dv))
    for s, (j0, j1) in enumerate(spans):
        if j1 <= j0:
            continue
        x = _scores(p, q[rows], rows, k, hq, j0, j1)
        ms = x.max(axis=1)                                                # max_l
        live = ms > NEG_INF
        e = np.exp(x - np.where(live, ms, 0.0)[:, None])
        e = np.where(live[:, None], e, 0.0)
        m[s], l[s], o[s] = ms, e.sum(axis=1), e @ v[j0:j1]                # sum_l, PV_l
    return m, l, o


def splitk_merge(m: np.ndarray, l: np.ndarray, o: np.ndarray):
    """Split-K global section WITHOUT the final divide (Fig. 5 ``s_max_global``,
    ``s_sum_global``; Eq. 8): M = max_s m_s, w_s = exp(m_s - M)
    (0 when m_s = -inf), L = sum w_s l_s, O = sum w_s O_s.
    Axis 0 indexes the parts. Returns the un-normalised triple (M, L, O)."""
    M = m.max(axis=0)                                                     # max_g
    live = M > NEG_INF
    Ms = np.where(live, M, 0.0)
    w = np.where(m > NEG_INF, np.exp(m - Ms[None]), 0.0)                  # repair exp(max_l - max_g)
    L = (w * l).sum(axis=0)                                               # sum_g
    O = (w[..., None] * o).sum(axis=0)
    return M, L, O


def splitk_combine(m: np.ndarray, l: np.ndarray, o: np.ndarray):
    """Eq. 8 combine followed by softmax_norm: returns (out, lse)."""
    M, L, O = splitk_merge(m, l, o)
    live = L > 0
    with np.errstate(invalid="ignore", divide="ignore"):
        out = np.where(live[..., None], O / L[..., None], 0.0)
        lse = np.where(live, M + np.log(L), NEG_INF)
    return out, lse
