"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO attention arithmetic. It only turns (seed, tensor id,
element index) into numbers, and converts bf16 bit patterns to wider floats.
Both sides of every parity test draw their inputs from here (or from the
bit-identical CUDA generator in ``datagen/gen.cu``), so neither side can
contaminate the other.

Generator (DESIGN.md §3 "input recipe"; a reading of SURVEY §8(c) Q14 and the
splitmix convention of SPEC S:571):

* ``key = mix64(seed * G + tensor_id)`` with ``G = 0x9E3779B97F4A7C15``;
* element ``i`` (flat, row-major over the tensor's logical shape) draws two
  64-bit words ``w_t = mix64(key + (2 i + t + 1) * G)``, ``t = 0, 1``;
* the eight 16-bit fields of ``w_0, w_1`` are summed (Irwin-Hall of 8 discrete
  uniforms), centred and scaled to unit variance in fp32:
  ``x = fp32(s - 4 * 65535) * fp32(1 / (65536 * sqrt(2/3)))`` (one correctly
  rounded fp32 multiply);
* bf16 tensors take ``x`` rounded to nearest-even.

Every step is integer arithmetic or a single IEEE-correctly-rounded fp32
operation, so the numpy path here and the CUDA path are bit-identical (tested
in ``tests/test_datagen.py`` and ``tests/test_gpu_parity.py``). The values are
approximately N(0, 1) with tails bounded at |x| <= sqrt(24) ~= 4.9.
"""
from __future__ import annotations

import numpy as np

G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
INV_SIGMA_F32 = np.float32(1.0 / (65536.0 * np.sqrt(2.0 / 3.0)))
CENTER = 4 * 65535

# Config seeds (SURVEY §8(d) "Synthetic inputs"): seed = 0x4E45505455 + 1000 * config_id.
SEED_BASE = 0x4E45505455
TENSOR_Q, TENSOR_K, TENSOR_V = 1, 2, 3


def config_seed(config_id: int) -> int:
    return SEED_BASE + 1000 * int(config_id)


def mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, tensor_id: int) -> int:
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) * G + np.uint64(tensor_id)
    return int(mix64(np.array([z], dtype=np.uint64))[0])


def _field_sum(w: np.ndarray) -> np.ndarray:
    m = np.uint64(0xFFFF)
    return ((w & m) + ((w >> np.uint64(16)) & m) + ((w >> np.uint64(32)) & m)
            + (w >> np.uint64(48))).astype(np.int64)


def normal_f32(key: int, start: int, count: int) -> np.ndarray:
    """fp32 values of flat elements [start, start + count) of stream ``key``."""
    out = np.empty(count, dtype=np.float32)
    chunk = 1 << 22
    k = np.uint64(key)
    for c0 in range(0, count, chunk):
        n = min(chunk, count - c0)
        idx = np.arange(start + c0, start + c0 + n, dtype=np.uint64)
        with np.errstate(over="ignore"):
            base = k + (np.uint64(2) * idx + np.uint64(1)) * G
            w0 = mix64(base)
            w1 = mix64(base + G)
        s = _field_sum(w0) + _field_sum(w1) - CENTER
        out[c0:c0 + n] = s.astype(np.float32) * INV_SIGMA_F32
    return out


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as uint16 bit patterns."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def tensor(seed: int, tensor_id: int, shape, dtype: str = "bf16", start: int = 0,
           count: int | None = None) -> np.ndarray:
    """Generate a full tensor (or a flat slice of it).

    dtype "bf16" / "f16" return uint16 bit patterns (RNE from the fp32 value),
    "f32" returns float32 values.
    The slice form lets the oracle regenerate any (b, h) slab of a tensor too
    large to materialise on the host.
    """
    n = int(np.prod(shape)) if count is None else int(count)
    x = normal_f32(stream_key(seed, tensor_id), start, n)
    if dtype == "bf16":
        x = f32_to_bf16_bits(x)
    elif dtype == "f16":
        x = x.astype(np.float16).view(np.uint16)      # IEEE round-to-nearest-even
    elif dtype != "f32":
        raise ValueError(f"unsupported dtype {dtype}")
    return x.reshape(shape) if count is None else x


def as_f64(x: np.ndarray, dtype: str) -> np.ndarray:
    """Exact fp64 view of generated values (bf16 bits or fp32)."""
    if dtype == "bf16":
        return bf16_bits_to_f32(x).astype(np.float64)
    if dtype == "f16":
        return np.asarray(x, dtype=np.uint16).view(np.float16).astype(np.float64)
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def _to_dtype(x32: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        return f32_to_bf16_bits(x32)
    if dtype == "f16":
        return x32.astype(np.float16).view(np.uint16)
    return x32.astype(np.float32)


def rising_rows(n: int) -> np.ndarray:
    """Rows that get the rising component in ``rising_logits`` (an irregular ~half of them,
    so a warp of 32 rows mixes rows that need the repair with rows that do not)."""
    i = np.arange(n, dtype=np.int64)
    return ((i * 37) >> 4) & 1 == 1


def rising_logits(q: np.ndarray, k: np.ndarray, dtype: str, amp: float, rate: float, tile: int = 128,
                  descending: bool = False):
    """Adversarial inputs for the repair tests: copies of generated q, k
    ([..., S, D], bits or fp32) with coordinate 0 replaced by
        q[..., i, 0] = amp if rising_rows(Sq)[i] else 0,
        k[..., j, 0] = rate * j / tile         (descending: rate * (Skv - 1 - j) / tile),
    each rounded to ``dtype``.  So q_i . k_j rises by about amp * rate along every `tile`
    keys of the ascending (or descending) KV walk and the running max of a rising row jumps
    by that much per KV tile.  No attention arithmetic: only the input values change."""
    q2, k2 = np.array(q, copy=True), np.array(k, copy=True)
    sq, skv = q.shape[-2], k.shape[-2]
    qa = np.where(rising_rows(sq), np.float32(amp), np.float32(0.0)).astype(np.float32)
    j = np.arange(skv, dtype=np.float64)
    if descending:
        j = (skv - 1) - j
    ka = (np.float64(rate) * j / tile).astype(np.float32)
    q2[..., 0] = _to_dtype(qa, dtype)
    k2[..., 0] = _to_dtype(ka, dtype)
    return q2, k2


def alibi_slopes(heads: int) -> np.ndarray:
    """Standard ALiBi slopes 2^(-8(h+1)/H), fp32."""
    h = np.arange(heads, dtype=np.float64)
    return np.exp2(-8.0 * (h + 1.0) / heads).astype(np.float32)


def slab(seed: int, tensor_id: int, shape, b: int, h: int, dtype: str = "bf16") -> np.ndarray:
    """The [S, D] slab at (b, h) of a contiguous [B, H, S, D] tensor."""
    B, H, S, D = shape
    start = ((b * H) + h) * S * D
    return tensor(seed, tensor_id, (B, H, S, D), dtype, start=start, count=S * D).reshape(S, D)
