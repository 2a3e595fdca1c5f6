"""The paper's motivating reduction chain (Fig. 2) on a [rows, cols]
matrix, written loop-for-loop in fp64 Python.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

* ``softmax_denominator``       -- Fig. 2a: s_max, s_exp, s_sum.
* ``softmax_denominator_naive_fused`` -- Fig. 2b: naive fusion,
  deliberately WRONG (reads xmax too early). Negative control.
* ``softmax_denominator_rolling`` -- Fig. 2c: repaired fusion
  with the repair term exp(xmax_0 - xmax_1). Also returns the per-iteration
  xsum trace so Eq. example-result can be checked.
* ``softmax_denominator_privatized`` -- Fig. 19.
* ``softmax_denominator_splitk`` -- Fig. 5.
* ``repair_h`` -- the solved repair function h(t, r, r') = exp(r - r') t
  (Fig. 18d).
"""
from __future__ import annotations

import math

import numpy as np


def repair_h(t, r, r_new):
    """h(t, r, r') = g(r', g_c^{-1}(r, t)) = exp(r - r') * t."""
    return np.exp(np.asarray(r, dtype=np.float64) - r_new) * t


def softmax_denominator(inp: np.ndarray) -> np.ndarray:
    """Fig. 2a: three separate loop nests."""
    rows, cols = inp.shape
    xmax = np.full(rows, -math.inf)
    for i in range(rows):
        for j in range(cols):                              # s_max
            xmax[i] = max(xmax[i], inp[i, j])
    xexp = np.empty_like(inp, dtype=np.float64)
    for i in range(rows):
        for j in range(cols):                              # s_exp
            xexp[i, j] = math.exp(inp[i, j] - xmax[i])
    xsum = np.zeros(rows)
    for i in range(rows):
        for j in range(cols):                              # s_sum
            xsum[i] += xexp[i, j]
    return xsum


def softmax_denominator_naive_fused(inp: np.ndarray) -> np.ndarray:
    """Fig. 2b: s_exp and s_sum naively fused under loop_j (incorrect)."""
    rows, cols = inp.shape
    xmax = np.full(rows, -math.inf)
    xsum = np.zeros(rows)
    for i in range(rows):
        for j in range(cols):
            xmax[i] = max(xmax[i], inp[i, j])
            xexp = math.exp(inp[i, j] - xmax[i])
            xsum[i] += xexp
    return xsum


def softmax_denominator_rolling(inp: np.ndarray, trace: bool = False):
    """Fig. 2c: the repaired single loop (Rolling Update output)."""
    rows, cols = inp.shape
    xsum = np.zeros(rows)
    hist = np.zeros((rows, cols))
    for i in range(rows):
        xmax_0 = -math.inf
        for j in range(cols):
            xmax_1 = max(xmax_0, inp[i, j])                                # s_max
            rep = math.exp(xmax_0 - xmax_1) if xmax_0 != -math.inf else 0.0
            xsum[i] = rep * xsum[i] + math.exp(inp[i, j] - xmax_1)         # s_sum, repaired
            xmax_0 = xmax_1
            hist[i, j] = xsum[i]
    return (xsum, hist) if trace else xsum


def softmax_denominator_privatized(inp: np.ndarray, split: int) -> np.ndarray:
    """Fig. 19: privatization (split ``split``) combined with rolling update."""
    rows, cols = inp.shape
    assert cols % split == 0
    xsum = np.zeros(rows)
    for i in range(rows):
        xmax_0 = -math.inf
        xmax_1 = -math.inf
        for j1 in range(cols // split):
            xmax_1p = -math.inf
            for j2 in range(split):                                        # max_local
                xmax_1p = max(xmax_1p, inp[i, j1 * split + j2])
            xmax_1 = max(xmax_1, xmax_1p)                                  # max_global
            xsump = 0.0
            for j2 in range(split):                                        # sum_local
                xsump += math.exp(inp[i, j1 * split + j2] - xmax_1)
            rep = math.exp(xmax_0 - xmax_1) if xmax_0 != -math.inf else 0.0
            xsum[i] = rep * xsum[i] + xsump
            xmax_0 = xmax_1
    return xsum


def softmax_denominator_splitk(inp: np.ndarray, split: int):
    """Fig. 5: local section over (i, j0) then the repaired global section.
    Returns (max_g, sum_g)."""
    rows, cols = inp.shape
    assert cols % split == 0
    nsplit = cols // split
    max_l = np.full((rows, nsplit), -math.inf)
    sum_l = np.zeros((rows, nsplit))
    for i in range(rows):
        for j0 in range(nsplit):
            for j1 in range(split):                                        # s_max_local
                max_l[i, j0] = max(max_l[i, j0], inp[i, j0 * split + j1])
            for j1 in range(split):                                        # s_sum_local
                sum_l[i, j0] += math.exp(inp[i, j0 * split + j1] - max_l[i, j0])
    max_g = np.full(rows, -math.inf)
    sum_g = np.zeros(rows)
    for i in range(rows):
        for j0 in range(nsplit):                                           # s_max_global
            max_g[i] = max(max_g[i], max_l[i, j0])
        for j0 in range(nsplit):                                           # s_sum_global
            sum_g[i] += math.exp(max_l[i, j0] - max_g[i]) * sum_l[i, j0]
    return max_g, sum_g


def softmax_rows(inp: np.ndarray):
    """Fig. 2a vectorised over rows in fp64 (the DEFINITION the softmax-rows
    kernel is checked against): xmax = max_j inp, xsum = sum_j exp(inp - xmax),
    plus the normalised softmax y = exp(inp - xmax) / xsum.  A row that is all
    -inf gives xmax = -inf, xsum = 0, y = 0 (reading R8)."""
    x = np.asarray(inp, dtype=np.float64)
    xmax = x.max(axis=1)
    live = xmax > -np.inf
    e = np.exp(x - np.where(live, xmax, 0.0)[:, None])            # s_exp, exp(-inf) = 0
    xsum = e.sum(axis=1)                                           # s_sum
    with np.errstate(invalid="ignore", divide="ignore"):
        y = np.where(live[:, None], e / np.where(live, xsum, 1.0)[:, None], 0.0)
    return xmax, xsum, y
