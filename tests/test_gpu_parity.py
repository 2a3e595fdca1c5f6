"""GPU parity: the CUDA path (through the C ABI via the thin binding) against
the fp64 oracle on the same seeded inputs.

Small shapes span several 128-row / 128-key tiles with ragged tails and are
compared element by element; BASELINE.json's full-size configs are run in the
same launch configuration bench.py times and compared on sampled rows the
oracle computes one by one."""
import math

import numpy as np
import pytest
import torch

import datagen
import oracle
from datagen import device as dgd
from tests.helpers import (FP32_MAX_ABS, LSE_TOL_BF16, LSE_TOL_FP32, assert_bf16_close, assert_lse_close, gen_qkv,
                           metrics, problem)

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2510_08726_b200 as pb


def _bf16_np(t: torch.Tensor) -> np.ndarray:
    return t.float().cpu().numpy().astype(np.float64)


def _kw_from(p: oracle.Problem, dev="cuda"):
    kw = dict(scale=p.scale, causal=p.causal, window=(p.window_left, p.window_right), softcap=p.softcap,
              kv_pos_offset=p.kv_pos_offset)
    if p.alibi_slopes is not None:
        kw["alibi_slopes"] = torch.tensor(np.asarray(p.alibi_slopes, dtype=np.float32), device=dev)
    if p.seqlen_kv_total is not None:
        kw["seqlen_kv_total"] = p.seqlen_kv_total
    if p.q_pos_offset is not None:
        kw["q_pos_offset"] = p.q_pos_offset
    return kw


# --------------------------------------------------------------------------- generator
def test_device_generator_is_bit_identical():
    for dt, tdt in (("bf16", torch.bfloat16), ("f32", torch.float32)):
        host = datagen.tensor(12345, 2, (3, 5, 77, 64), dt)
        dev = dgd.tensor(12345, 2, (3, 5, 77, 64), tdt).cpu()
        if dt == "bf16":
            np.testing.assert_array_equal(dev.view(torch.int16).numpy().view(np.uint16), host)
        else:
            np.testing.assert_array_equal(dev.numpy(), host)


# --------------------------------------------------------------------------- fp32 SIMT path
FP32_CASES = [
    dict(B=1, Hq=1, Hkv=1, S=64, D=16),                                   # config 1 (tiny)
    dict(B=2, Hq=4, Hkv=2, S=70, D=40, causal=True),
    dict(B=1, Hq=2, Hkv=1, S=45, D=64, alibi=True, causal=True),
    dict(B=1, Hq=2, Hkv=2, S=50, D=128, softcap=2.0, causal=True),
    dict(B=1, Hq=2, Hkv=2, S=65, D=256, window=(9, 3)),
]


@pytest.mark.parametrize("case", range(len(FP32_CASES)))
def test_fp32_forward(case):
    c = dict(FP32_CASES[case])
    B, Hq, Hkv, S, D = c.pop("B"), c.pop("Hq"), c.pop("Hkv"), c.pop("S"), c.pop("D")
    kw = {}
    if c.pop("alibi", False):
        kw["alibi_slopes"] = datagen.alibi_slopes(Hq)
    if "window" in c:
        kw["window_left"], kw["window_right"] = c.pop("window")
    kw.update(c)
    p = problem(B, Hq, Hkv, S, S, D, **kw)
    raw, f64 = gen_qkv(datagen.config_seed(1) + case, B, Hq, Hkv, S, S, D, "f32")
    ref_o, ref_l = oracle.attention(p, *f64)
    q, k, v = (dgd.to_device(x) for x in raw)
    o, lse = pb.fused_fwd(q, k, v, return_lse=True, **_kw_from(p))
    err = np.abs(o.cpu().numpy().astype(np.float64) - ref_o).max()
    assert err <= FP32_MAX_ABS, err
    assert_lse_close(lse.cpu().numpy(), ref_l, LSE_TOL_FP32, "fp32 lse")


# --------------------------------------------------------------------------- bf16 tcgen05 prefill, small shapes
VARIANTS = {
    "global": dict(),
    "causal": dict(causal=True),
    "window_causal": dict(causal=True, window_left=37),
    "window_band": dict(window_left=150, window_right=21),
    "alibi_causal": dict(causal=True, alibi=True),
    "softcap_causal": dict(causal=True, softcap=2.0),
    "alibi_softcap": dict(alibi=True, softcap=2.0, window_left=200, window_right=0),
    # D = 64 folds ALiBi into the QK contraction: tiles wholly below, wholly above and across
    # the diagonal take different paths (fwd_tc.cu ext_class)
    "alibi": dict(alibi=True),
    "alibi_band": dict(alibi=True, window_left=150, window_right=21),
    # cap 8: |x / cap| <= 1/2 for most warps (tanh on the FMA pipe for every other column),
    # above it for some (all on the SFU) -- both paths in one launch
    "softcap8_causal": dict(causal=True, softcap=8.0),
}


@pytest.mark.parametrize("D", [128, 64])
@pytest.mark.parametrize("name", list(VARIANTS))
def test_bf16_prefill_small(name, D):
    kw = dict(VARIANTS[name])
    B, Hq, Hkv, S = 2, 4, 2, 333           # 2 q-blocks of 256 rows, 3 KV tiles, ragged tails
    if kw.pop("alibi", False):
        kw["alibi_slopes"] = datagen.alibi_slopes(Hq)
    p = problem(B, Hq, Hkv, S, S, D, **kw)
    raw, f64 = gen_qkv(77 + D, B, Hq, Hkv, S, S, D)
    ref_o, ref_l = oracle.attention(p, *f64)
    q, k, v = (dgd.to_device(x) for x in raw)
    o, lse = pb.fused_fwd(q, k, v, return_lse=True, **_kw_from(p))
    torch.cuda.synchronize()
    assert pb.last_launch_count() == 1
    assert_bf16_close(_bf16_np(o), ref_o, f"{name} D={D}")
    assert_lse_close(lse.cpu().numpy(), ref_l, LSE_TOL_BF16, f"{name} D={D} lse")


@pytest.mark.parametrize("Sq,Skv,extra", [
    (100, 700, dict(causal=True)),                                   # chunked prefill, bottom-right
    (1, 513, dict(causal=True)),                                     # decode shape through prefill kernel
    (300, 64, dict(causal=True)),                                    # Sq > Skv: leading rows fully masked
    (257, 300, dict(causal=True, kv_pos_offset=100, seqlen_kv_total=400)),  # KV shard of a longer sequence
    (130, 1000, dict(window_left=60, window_right=60, q_pos_offset=400)),   # band in the middle
    (129, 129, dict()),
])
def test_bf16_prefill_rectangular(Sq, Skv, extra):
    _rectangular(Sq, Skv, extra, 128)


@pytest.mark.parametrize("Sq,Skv,extra", [
    (130, 1000, dict(q_pos_offset=400)),                                   # keys on both sides, non-causal
    (257, 300, dict(causal=True, kv_pos_offset=100, seqlen_kv_total=400)), # KV shard of a longer sequence
    (100, 700, dict(causal=True)),                                         # chunked prefill, bottom-right
    (300, 900, dict(window_left=70, window_right=300, q_pos_offset=250)),  # band crossing tile edges
    (200, 600, dict(scale=1e-3)),                                          # |slope / scale| = 707: large ALiBi term
])
@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("D", [64, 128])
def test_alibi_rectangular(Sq, Skv, extra, dtype, D):
    """ALiBi by tile class: D = 64 folds the bias into the QK contraction (fp16 with |s| >= 256
    falls back); D = 128 uses the linear form on tiles of uniform sign; both fix up mixed tiles."""
    _rectangular(Sq, Skv, dict(extra, alibi_slopes=datagen.alibi_slopes(4)), D, Hq=4, Hkv=2, dtype=dtype)


def _rectangular(Sq, Skv, extra, D, Hq=2, Hkv=1, dtype="bf16"):
    B = 1
    p = problem(B, Hq, Hkv, Sq, Skv, D, **extra)
    gdt = "f16" if dtype == "fp16" else "bf16"
    raw, f64 = gen_qkv(1000 + Sq + Skv + D, B, Hq, Hkv, Sq, Skv, D, gdt)
    ref_o, ref_l = oracle.attention(p, *f64)
    q, k, v = (dgd.to_device(x, dtype=gdt) for x in raw)
    o, lse = pb.fused_fwd(q, k, v, return_lse=True, **_kw_from(p))
    assert_bf16_close(_bf16_np(o), ref_o, f"{dtype} D={D} Sq={Sq} Skv={Skv} {extra}")
    assert_lse_close(lse.cpu().numpy(), ref_l, LSE_TOL_BF16, "lse")


SPLIT_CASES = [   # (B, Hq, Hkv, Sq, Skv, D, splits, variant)
    (1, 4, 2, 16, 2048, 128, 4, dict()),                                   # Table 3 corner, GQA
    (1, 2, 2, 100, 1000, 128, 3, dict(causal=True)),                       # chunked prefill, ragged
    (2, 2, 1, 300, 1300, 64, 5, dict(causal=True, alibi=True)),            # 2 q-blocks, D = 64
    (1, 2, 2, 64, 777, 128, 6, dict(softcap=2.0)),
    (1, 2, 1, 200, 1500, 128, 4, dict(window_left=300, window_right=0, causal=True)),   # empty splits
    (1, 2, 2, 129, 900, 128, 7, dict(causal=True, kv_pos_offset=100, seqlen_kv_total=1000)),
]


@pytest.mark.parametrize("case", range(len(SPLIT_CASES)))
def test_prefill_kv_split(case):
    """NEXT-2: the KV axis split across CTAs (normalised partials + Eq. 8 merge) equals the
    oracle, and the unsplit kernel within tolerance; 2 launches."""
    B, Hq, Hkv, Sq, Skv, D, splits, var = SPLIT_CASES[case]
    var = dict(var)
    if var.pop("alibi", False):
        var["alibi_slopes"] = datagen.alibi_slopes(Hq)
    p = problem(B, Hq, Hkv, Sq, Skv, D, **var)
    raw, f64 = gen_qkv(1500 + case, B, Hq, Hkv, Sq, Skv, D)
    ref_o, ref_l = oracle.attention(p, *f64)
    q, k, v = (dgd.to_device(x) for x in raw)
    o, lse = pb.fused_fwd(q, k, v, return_lse=True, kv_splits=splits, **_kw_from(p))
    torch.cuda.synchronize()
    assert pb.last_launch_count() == 2
    assert_bf16_close(_bf16_np(o), ref_o, f"split case {case}")
    assert_lse_close(lse.cpu().numpy(), ref_l, LSE_TOL_BF16, f"split case {case} lse")
    o1 = pb.fused_fwd(q, k, v, kv_splits=1, **_kw_from(p))
    torch.cuda.synchronize()
    assert pb.last_launch_count() == 1
    assert (o1.float() - o.float()).abs().max().item() <= 2e-2
    # strided output view (the merge writes a [B][H][Sq][D] view with arbitrary strides)
    big = torch.zeros(B, Hq, Sq + 3, D + 64, dtype=q.dtype, device="cuda")
    pb.fused_fwd(q, k, v, out=big[:, :, 1:Sq + 1, 32:32 + D], kv_splits=splits, **_kw_from(p))
    torch.cuda.synchronize()
    assert torch.equal(big[:, :, 1:Sq + 1, 32:32 + D], o)
    assert big[:, :, 0].abs().max().item() == 0 and big[..., :32].abs().max().item() == 0


def test_prefill_kv_split_fp16_auto():
    """Auto split on a small grid (B*Hq*qblocks << SMs), fp16."""
    B, Hq, Hkv, Sq, Skv, D = 1, 8, 8, 32, 2048, 128
    p = problem(B, Hq, Hkv, Sq, Skv, D, causal=True)
    raw, f64 = gen_qkv(1600, B, Hq, Hkv, Sq, Skv, D, dtype="f16")
    ref_o, _ = oracle.attention(p, *f64)
    q, k, v = (dgd.to_device(x, dtype="f16") for x in raw)
    o = pb.fused_fwd(q, k, v, **_kw_from(p))
    torch.cuda.synchronize()
    assert pb.last_launch_count() == 2          # the default split kicked in
    assert o.dtype == torch.float16
    assert_bf16_close(_bf16_np(o), ref_o, "fp16 auto split")


def test_bf16_prefill_strided_views_and_determinism():
    """Non-contiguous (sliced) q/k/v views and bitwise run-to-run determinism."""
    B, Hq, Hkv, S, D = 2, 4, 4, 300, 128
    p = problem(B, Hq, Hkv, S, S, D, causal=True)
    raw, f64 = gen_qkv(4242, B, Hq, Hkv, S, S, D)
    ref_o, _ = oracle.attention(p, *f64)
    big = [torch.zeros(B, Hq + 2, S + 16, D, dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    views = []
    for t, x in zip(big, raw):
        t[:, 1:Hq + 1, 8:S + 8] = dgd.to_device(x)
        views.append(t[:, 1:Hq + 1, 8:S + 8])
    o1 = pb.fused_fwd(*views, causal=True)
    o2 = pb.fused_fwd(*views, causal=True)
    assert torch.equal(o1, o2)
    assert_bf16_close(_bf16_np(o1), ref_o, "strided")


# --------------------------------------------------------------------------- full-size configs, sampled rows
FULL = {
    "mha_noncausal": dict(cid=2, B=8, Hq=16, Hkv=16, S=4096, D=128),
    "mha_causal": dict(cid=2, B=8, Hq=16, Hkv=16, S=4096, D=128, causal=True),
    "gqa_window": dict(cid=3, B=4, Hq=32, Hkv=8, S=8192, D=128, causal=True, window_left=4095),
    "variants_scaled_dot": dict(cid=4, B=8, Hq=16, Hkv=16, S=2048, D=64),
    "variants_alibi_causal": dict(cid=4, B=8, Hq=16, Hkv=16, S=2048, D=64, causal=True, alibi=True),
    "variants_alibi": dict(cid=4, B=8, Hq=16, Hkv=16, S=2048, D=64, alibi=True),
    "mha_alibi_causal": dict(cid=2, B=8, Hq=16, Hkv=16, S=4096, D=128, causal=True, alibi=True),
    "variants_softcap_causal": dict(cid=4, B=8, Hq=16, Hkv=16, S=2048, D=64, causal=True, softcap=2.0),
    "variants_softcap50_causal": dict(cid=4, B=8, Hq=16, Hkv=16, S=2048, D=64, causal=True, softcap=50.0),
}


def _sample_rows(S, rng, n=40):
    fixed = [0, 1, 127, 128, 255, 256, S // 2, S - 129, S - 128, S - 2, S - 1]
    return sorted(set([r for r in fixed if 0 <= r < S] + list(rng.integers(0, S, n))))


@pytest.mark.parametrize("name", list(FULL))
def test_bf16_prefill_full_config_sampled(name):
    c = dict(FULL[name])
    cid, B, Hq, Hkv, S, D = (c.pop(k) for k in ("cid", "B", "Hq", "Hkv", "S", "D"))
    if c.pop("alibi", False):
        c["alibi_slopes"] = datagen.alibi_slopes(Hq)
    p = problem(B, Hq, Hkv, S, S, D, **c)
    seed = datagen.config_seed(cid)
    q = dgd.tensor(seed, datagen.TENSOR_Q, (B, Hq, S, D))
    k = dgd.tensor(seed, datagen.TENSOR_K, (B, Hkv, S, D))
    v = dgd.tensor(seed, datagen.TENSOR_V, (B, Hkv, S, D))
    o, lse = pb.fused_fwd(q, k, v, return_lse=True, **_kw_from(p))
    torch.cuda.synchronize()
    rng = np.random.default_rng(cid)
    pairs = sorted({(0, 0), (B - 1, Hq - 1), (int(rng.integers(B)), int(rng.integers(Hq)))})
    got, ref, lg, lr = [], [], [], []
    for b, hq in pairs:
        g = oracle.head_group(p, hq)
        qs = datagen.as_f64(datagen.slab(seed, datagen.TENSOR_Q, (B, Hq, S, D), b, hq), "bf16")
        ks = datagen.as_f64(datagen.slab(seed, datagen.TENSOR_K, (B, Hkv, S, D), b, g), "bf16")
        vs = datagen.as_f64(datagen.slab(seed, datagen.TENSOR_V, (B, Hkv, S, D), b, g), "bf16")
        rows = _sample_rows(S, rng)
        ro, rl = oracle.attention_bh(p, qs, ks, vs, hq, rows=rows)
        got.append(_bf16_np(o[b, hq, rows]))
        ref.append(ro)
        lg.append(lse[b, hq, rows].cpu().numpy())
        lr.append(rl)
    assert_bf16_close(np.concatenate(got), np.concatenate(ref), name)
    assert_lse_close(np.concatenate(lg), np.concatenate(lr), LSE_TOL_BF16, name + " lse")


# --------------------------------------------------------------------------- decode (Split-K Update)
def _split_bounds(Skv, splits):
    per = -(-Skv // splits)
    L = 64 * (-(-per // 64))
    return [min(s * L, Skv) for s in range(splits)] + [Skv]


DECODE_CASES = [
    dict(B=2, Hq=8, Hkv=2, Skv=1000, D=128, splits=1),
    dict(B=2, Hq=8, Hkv=2, Skv=1000, D=128, splits=3),
    dict(B=2, Hq=8, Hkv=2, Skv=1000, D=128, splits=7),
    dict(B=2, Hq=8, Hkv=2, Skv=1000, D=128, splits=40),       # more splits than 64-key stages: empty parts
    dict(B=1, Hq=4, Hkv=4, Skv=777, D=128, splits=5),         # MHA (G = 1)
    dict(B=1, Hq=16, Hkv=2, Skv=517, D=64, splits=4),         # G = 8, D = 64
    dict(B=3, Hq=8, Hkv=2, Skv=300, D=128, splits=2, alibi=True, causal=True),
    dict(B=1, Hq=8, Hkv=2, Skv=300, D=128, splits=2, softcap=2.0),
    dict(B=1, Hq=8, Hkv=2, Skv=600, D=128, splits=4, window_left=200, causal=True),
]


@pytest.mark.parametrize("case", range(len(DECODE_CASES)))
def test_decode_parts_and_output(case):
    c = dict(DECODE_CASES[case])
    B, Hq, Hkv, Skv, D, splits = (c.pop(k) for k in ("B", "Hq", "Hkv", "Skv", "D", "splits"))
    if c.pop("alibi", False):
        c["alibi_slopes"] = datagen.alibi_slopes(Hq)
    p = problem(B, Hq, Hkv, 1, Skv, D, **c)
    raw, (q64, k64, v64) = gen_qkv(500 + case, B, Hq, Hkv, 1, Skv, D)
    ref_o, ref_l = oracle.attention(p, q64, k64, v64)
    q, k, v = (dgd.to_device(x) for x in raw)
    parts = pb.Parts.empty(splits, B, Hq, D, "cuda")
    o, lse = pb.splitkv_decode(q, k, v, num_splits=splits, parts=parts, return_lse=True, **_kw_from(p))
    torch.cuda.synchronize()
    assert pb.last_launch_count() == 2
    assert_bf16_close(_bf16_np(o), ref_o, f"decode case {case}")
    assert_lse_close(lse.cpu().numpy(), ref_l[:, :, 0], LSE_TOL_BF16, "decode lse")
    # the local-section triples themselves (Fig. 5 max_l, sum_l, PV_l)
    bounds = _split_bounds(Skv, splits)
    gm, gl, go = parts.m.cpu().numpy(), parts.l.cpu().numpy(), parts.o.cpu().numpy()
    for b in range(B):
        for hq in range(Hq):
            g = oracle.head_group(p, hq)
            m, l, po = oracle.splitk_local_bh(p, q64[b, hq], k64[b, g], v64[b, g], hq, bounds)
            fin = np.isfinite(m[:, 0])
            assert np.array_equal(np.isfinite(gm[:, b, hq]), fin)
            np.testing.assert_allclose(gm[fin, b, hq], m[fin, 0], atol=2e-3)
            np.testing.assert_allclose(gl[:, b, hq], l[:, 0], rtol=1e-2, atol=1e-3)
            assert metrics(go[:, b, hq], po[:, 0])[1] < 5e-3


@pytest.mark.parametrize("B", [1, 4, 8, 16])
def test_decode_full_config_sampled(B):
    """Config 5: Hq=32, Hkv=8, KV 128K, D=128, causal (all keys), auto splits -- the split
    count bench.py times (B >= 8: >= 64 (b, hkv) groups, so the count rounds up to <= 2
    CTAs per SM, csrc/api.cu attn_splitkv_default_splits)."""
    Hq, Hkv, L, D = 32, 8, 131072, 128
    p = problem(B, Hq, Hkv, 1, L, D, causal=True)
    seed = datagen.config_seed(5)
    q = dgd.tensor(seed, datagen.TENSOR_Q, (B, Hq, 1, D))
    k = dgd.tensor(seed, datagen.TENSOR_K, (B, Hkv, L, D))
    v = dgd.tensor(seed, datagen.TENSOR_V, (B, Hkv, L, D))
    o, lse = pb.splitkv_decode(q, k, v, causal=True, return_lse=True)
    torch.cuda.synchronize()
    rng = np.random.default_rng(B)
    got, ref = [], []
    for b, g in sorted({(0, 0), (B - 1, Hkv - 1), (int(rng.integers(B)), int(rng.integers(Hkv)))}):
        ks = datagen.as_f64(datagen.slab(seed, datagen.TENSOR_K, (B, Hkv, L, D), b, g), "bf16")
        vs = datagen.as_f64(datagen.slab(seed, datagen.TENSOR_V, (B, Hkv, L, D), b, g), "bf16")
        for hq in range(g * 4, g * 4 + 4):
            qs = datagen.as_f64(datagen.slab(seed, datagen.TENSOR_Q, (B, Hq, 1, D), b, hq), "bf16")
            ro, rl = oracle.attention_bh(p, qs, ks, vs, hq)
            got.append(_bf16_np(o[b, hq]))
            ref.append(ro)
            assert abs(lse[b, hq].item() - rl[0]) <= LSE_TOL_BF16
    assert_bf16_close(np.concatenate(got), np.concatenate(ref), f"decode B={B}")


@pytest.mark.parametrize("case", range(len(DECODE_CASES)))
def test_decode_fused_combine(case):
    """parts=None: the Eq. 8 global section runs inside the split kernel (last CTA per
    (b, hkv) combines, one launch).  Same output as the two-launch path, equal to the
    oracle, and the ticket block is back to zero after every call (include/attn.h)."""
    c = dict(DECODE_CASES[case])
    B, Hq, Hkv, Skv, D, splits = (c.pop(k) for k in ("B", "Hq", "Hkv", "Skv", "D", "splits"))
    if c.pop("alibi", False):
        c["alibi_slopes"] = datagen.alibi_slopes(Hq)
    p = problem(B, Hq, Hkv, 1, Skv, D, **c)
    raw, (q64, k64, v64) = gen_qkv(500 + case, B, Hq, Hkv, 1, Skv, D)
    ref_o, ref_l = oracle.attention(p, q64, k64, v64)
    q, k, v = (dgd.to_device(x) for x in raw)
    kw = _kw_from(p)
    ws = torch.zeros(pb.workspace_bytes(q, k, splits), dtype=torch.uint8, device="cuda")
    outs = []
    for _ in range(3):   # the same workspace three times: tickets must reset
        o, lse = pb.splitkv_decode(q, k, v, num_splits=splits, workspace=ws, return_lse=True, **kw)
        torch.cuda.synchronize()
        assert pb.last_launch_count() == 1
        outs.append(o.clone())
        tickets = ws[:(B * Hkv * 4 + 255) // 256 * 256]
        assert int(tickets.count_nonzero()) == 0
    assert_bf16_close(_bf16_np(outs[0]), ref_o, f"fused decode case {case}")
    assert_lse_close(lse.cpu().numpy(), ref_l[:, :, 0], LSE_TOL_BF16, "fused decode lse")
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    parts = pb.Parts.empty(splits, B, Hq, D, "cuda")
    o2 = pb.splitkv_decode(q, k, v, num_splits=splits, parts=parts, **kw)   # two-launch path
    torch.cuda.synchronize()
    assert (o2.float() - outs[0].float()).abs().max().item() <= 2 ** -7


MULTI_CASES = [   # (B, Hq, Hkv, Sq, Skv, D, variant, dtype)
    (2, 8, 2, 2, 1000, 128, dict(causal=True), "bf16"),                 # G*Sq = 8: low mma rows only
    (2, 8, 2, 4, 1000, 128, dict(causal=True), "bf16"),                 # 16 rows: both row halves
    (1, 4, 4, 16, 777, 128, dict(causal=True), "bf16"),                 # MHA, 16 queries
    (1, 16, 2, 2, 600, 64, dict(causal=True, alibi=True), "bf16"),      # G = 8, D = 64
    (1, 8, 2, 3, 900, 128, dict(causal=True, window_left=300), "f16"),  # 12 rows, window, fp16
    (1, 16, 1, 1, 500, 128, dict(softcap=2.0), "bf16"),                 # G = 16 single query
]


@pytest.mark.parametrize("case", range(len(MULTI_CASES)))
def test_decode_multi_token(case):
    """NEXT-2 small s_q: the G * s_q (head, query) rows of a KV group packed into one
    16-row mma tile of the split-KV decode kernel, per-row causal masks, fused combine."""
    B, Hq, Hkv, Sq, Skv, D, var, dt = MULTI_CASES[case]
    var = dict(var)
    if var.pop("alibi", False):
        var["alibi_slopes"] = datagen.alibi_slopes(Hq)
    p = problem(B, Hq, Hkv, Sq, Skv, D, **var)
    raw, f64 = gen_qkv(1700 + case, B, Hq, Hkv, Sq, Skv, D, dtype=dt)
    ref_o, ref_l = oracle.attention(p, *f64)
    q, k, v = (dgd.to_device(x, dtype=dt) for x in raw)
    for splits in (0, 3):
        o, lse = pb.splitkv_decode(q, k, v, num_splits=splits, return_lse=True, **_kw_from(p))
        torch.cuda.synchronize()
        assert pb.last_launch_count() == 1
        assert o.shape == q.shape
        assert_bf16_close(_bf16_np(o), ref_o, f"multi-token decode case {case} splits={splits}")
        got_l = lse.cpu().numpy().reshape(ref_l.shape)
        assert_lse_close(got_l, ref_l, LSE_TOL_BF16, f"multi-token decode lse {case}")


def test_combine_kernel_matches_oracle():
    """attn_combine alone on oracle-made partials, with empty (-inf) parts and
    an un-normalised acc output merged again (hierarchical, R3)."""
    P, B, H, D = 9, 2, 3, 128
    rng = np.random.default_rng(9)
    m = rng.standard_normal((P, B, H)) * 3
    m[2] = -np.inf
    m[5, 0, 1] = -np.inf
    l = np.where(np.isfinite(m), rng.uniform(0.5, 30, (P, B, H)), 0.0)
    o = rng.standard_normal((P, B, H, D)) * l[..., None]
    ref_o, ref_l = oracle.splitk_combine(m, l, o)
    parts = pb.Parts(*(torch.tensor(x, dtype=torch.float32, device="cuda") for x in (m, l, o)))
    out, lse = pb.combine(parts, out_dtype=torch.float32, return_lse=True)
    np.testing.assert_allclose(out[:, :, 0].cpu().numpy(), ref_o, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(lse.cpu().numpy(), ref_l, rtol=1e-5, atol=1e-5)
    # two-level merge: parts [0,4) and [4,9) -> acc triples -> combine again
    accs = []
    for sl in (slice(0, 4), slice(4, 9)):
        acc = pb.Parts.empty(1, B, H, D, "cuda")
        pb.combine(pb.Parts(parts.m[sl], parts.l[sl], parts.o[sl]), acc=acc, want_out=False)
        accs.append(acc)
    two = pb.Parts(torch.cat([a.m for a in accs]), torch.cat([a.l for a in accs]), torch.cat([a.o for a in accs]))
    out2 = pb.combine(two, out_dtype=torch.float32)
    np.testing.assert_allclose(out2[:, :, 0].cpu().numpy(), ref_o, rtol=1e-5, atol=1e-5)


def test_host_buffers_end_to_end():
    """The e2e path: pinned host tensors in, host tensor out."""
    B, Hq, Hkv, S, D = 1, 2, 2, 200, 128
    p = problem(B, Hq, Hkv, S, S, D, causal=True)
    raw, f64 = gen_qkv(31337, B, Hq, Hkv, S, S, D)
    ref_o, _ = oracle.attention(p, *f64)
    host = [dgd.to_device(x, "cpu").pin_memory() for x in raw]
    o = pb.fused_fwd(*host, causal=True)
    assert o.device.type == "cpu"
    assert_bf16_close(o.float().numpy().astype(np.float64), ref_o, "host e2e")


def test_host_buffers_pipelined_chunks():
    """The e2e path cuts the batch into chunks over two streams (copies overlap the kernel):
    the result must equal the device call bit for bit, lse included, pinned or not."""
    B, Hq, Hkv, S, D = 5, 4, 2, 300, 128
    p = problem(B, Hq, Hkv, S, S, D, causal=True, alibi_slopes=datagen.alibi_slopes(Hq))
    raw, f64 = gen_qkv(31338, B, Hq, Hkv, S, S, D)
    ref_o, ref_l = oracle.attention(p, *f64)
    dev = [dgd.to_device(x) for x in raw]
    slopes = torch.tensor(np.asarray(p.alibi_slopes, dtype=np.float32))
    o_dev, l_dev = pb.fused_fwd(*dev, causal=True, alibi_slopes=slopes.cuda(), return_lse=True)
    for pinned in (True, False):
        host = [t.cpu().pin_memory() if pinned else t.cpu() for t in dev]
        o, l = pb.fused_fwd(*host, causal=True, alibi_slopes=slopes, return_lse=True)
        assert o.device.type == "cpu" and l.device.type == "cpu"
        assert torch.equal(o, o_dev.cpu()) and torch.equal(l, l_dev.cpu())
    assert_bf16_close(o.float().numpy().astype(np.float64), ref_o, "host e2e chunks")
    assert_lse_close(l.numpy(), ref_l, LSE_TOL_BF16, "host e2e lse")


# --------------------------------------------------------------------------- fp16 inputs (NEXT-1, the paper's precision P:946)
def test_device_generator_fp16_is_bit_identical():
    host = datagen.tensor(999, 3, (2, 3, 50, 64), "f16")
    dev = dgd.tensor(999, 3, (2, 3, 50, 64), torch.float16).cpu()
    np.testing.assert_array_equal(dev.view(torch.int16).numpy().view(np.uint16), host)


@pytest.mark.parametrize("D", [128, 64])
@pytest.mark.parametrize("name", ["global", "causal", "alibi_causal", "softcap_causal", "window_band", "alibi",
                                  "softcap8_causal"])
def test_fp16_prefill_small(name, D):
    kw = dict(VARIANTS[name])
    B, Hq, Hkv, S = 1, 4, 2, 300
    if kw.pop("alibi", False):
        kw["alibi_slopes"] = datagen.alibi_slopes(Hq)
    p = problem(B, Hq, Hkv, S, S, D, **kw)
    raw, f64 = gen_qkv(4000 + D, B, Hq, Hkv, S, S, D, "f16")
    ref_o, ref_l = oracle.attention(p, *f64)
    q, k, v = (dgd.to_device(x, dtype="f16") for x in raw)
    o, lse = pb.fused_fwd(q, k, v, return_lse=True, **_kw_from(p))
    assert o.dtype == torch.float16
    assert_bf16_close(o.float().cpu().numpy().astype(np.float64), ref_o, f"fp16 {name} D={D}")
    assert_lse_close(lse.cpu().numpy(), ref_l, LSE_TOL_BF16, "fp16 lse")


@pytest.mark.parametrize("case", [0, 2, 6])
def test_fp16_decode(case):
    c = dict(DECODE_CASES[case])
    B, Hq, Hkv, Skv, D, splits = (c.pop(k) for k in ("B", "Hq", "Hkv", "Skv", "D", "splits"))
    if c.pop("alibi", False):
        c["alibi_slopes"] = datagen.alibi_slopes(Hq)
    p = problem(B, Hq, Hkv, 1, Skv, D, **c)
    raw, f64 = gen_qkv(5000 + case, B, Hq, Hkv, 1, Skv, D, "f16")
    ref_o, _ = oracle.attention(p, *f64)
    q, k, v = (dgd.to_device(x, dtype="f16") for x in raw)
    o = pb.splitkv_decode(q, k, v, num_splits=splits, **_kw_from(p))
    assert o.dtype == torch.float16
    assert_bf16_close(o.float().cpu().numpy().astype(np.float64), ref_o, f"fp16 decode {case}")
