"""Shared test helpers: seeded inputs (datagen), oracle calls, error metrics.

Tolerances (BASELINE.json north_star): bf16 max|err| <= 2e-2
and relative RMS <= 5e-3; fp32 max|err| <= 1e-4.  lse: |err| <= 2e-3 (bf16
inputs; derived in DESIGN.md §5), 1e-4 (fp32)."""
from __future__ import annotations

import math

import numpy as np

import datagen
import oracle

BF16_MAX_ABS = 2e-2
BF16_REL_RMS = 5e-3
FP32_MAX_ABS = 1e-4
LSE_TOL_BF16 = 2e-3
LSE_TOL_FP32 = 1e-4


def gen_qkv(seed, B, Hq, Hkv, Sq, Skv, D, dtype="bf16"):
    """Host copies of the inputs: raw (bf16 bits or fp32) and exact fp64."""
    q = datagen.tensor(seed, datagen.TENSOR_Q, (B, Hq, Sq, D), dtype)
    k = datagen.tensor(seed, datagen.TENSOR_K, (B, Hkv, Skv, D), dtype)
    v = datagen.tensor(seed, datagen.TENSOR_V, (B, Hkv, Skv, D), dtype)
    return (q, k, v), tuple(datagen.as_f64(x, dtype) for x in (q, k, v))


def metrics(gpu: np.ndarray, ref: np.ndarray):
    err = np.abs(gpu.astype(np.float64) - ref)
    max_abs = float(err.max()) if err.size else 0.0
    den = math.sqrt(float((ref ** 2).sum()))
    rel_rms = math.sqrt(float((err ** 2).sum())) / den if den > 0 else 0.0
    return max_abs, rel_rms


def assert_bf16_close(gpu: np.ndarray, ref: np.ndarray, what: str = ""):
    max_abs, rel_rms = metrics(gpu, ref)
    floor_abs, floor_rms = metrics(datagen.bf16_bits_to_f32(datagen.f32_to_bf16_bits(ref.astype(np.float32))), ref)
    msg = (f"{what}: max_abs={max_abs:.3e} rel_rms={rel_rms:.3e} "
           f"(ideal bf16 floor {floor_abs:.3e}/{floor_rms:.3e})")
    if max_abs > BF16_MAX_ABS or rel_rms > BF16_REL_RMS:
        idx = np.unravel_index(np.argmax(np.abs(gpu - ref)), ref.shape)
        msg += f" worst at {idx}: gpu={gpu[idx]} ref={ref[idx]}"
        raise AssertionError(msg)
    return max_abs, rel_rms


def assert_lse_close(gpu: np.ndarray, ref: np.ndarray, tol: float, what: str = ""):
    fin = np.isfinite(ref)
    assert np.array_equal(np.isfinite(gpu), fin), f"{what}: -inf pattern of lse differs"
    if fin.any():
        err = np.abs(gpu[fin] - ref[fin]).max()
        assert err <= tol, f"{what}: lse max err {err:.3e} > {tol}"


def problem(B, Hq, Hkv, Sq, Skv, D, **kw):
    return oracle.Problem(B, Hq, Hkv, Sq, Skv, D, scale=kw.pop("scale", 1.0 / math.sqrt(D)), **kw)


def oracle_full(p, q64, k64, v64):
    return oracle.attention(p, q64, k64, v64)
