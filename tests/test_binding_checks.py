"""The Python binding's argument checks: shapes, dtypes and devices the C ABI
cannot see (it gets pointers and strides, not allocation sizes) are rejected with
ValueError before anything is launched.  CPU-only: 'meta' tensors carry shapes and
dtypes without memory, so nothing here touches a GPU."""
import pytest
import torch

import paper_2510_08726_b200 as pb

M = "meta"


def t(*shape, dtype=torch.bfloat16):
    return torch.empty(*shape, dtype=dtype, device=M)


def qkv(B=1, Hq=4, Hkv=2, Sq=64, Skv=64, D=128):
    return t(B, Hq, Sq, D), t(B, Hkv, Skv, D), t(B, Hkv, Skv, D)


@pytest.mark.parametrize("bad,match", [
    (dict(v=t(1, 2, 63, 128)), "v .* must have k's shape"),
    (dict(k=t(1, 2, 64, 128, dtype=torch.float32), v=t(1, 2, 64, 128, dtype=torch.float32)), "dtype"),
    (dict(v=t(1, 2, 64, 128, dtype=torch.float16)), "dtype"),
    (dict(out=t(1, 4, 32, 128)), "out .* must have q's shape"),
    (dict(out=t(1, 4, 64, 128, dtype=torch.float16)), "dtype"),
    (dict(lse=torch.empty(1, 4, 32, device=M)), "lse must have shape"),
    (dict(lse=torch.empty(1, 4, 64, device=M, dtype=torch.float64)), "float32"),
    (dict(k=t(1, 3, 64, 128), v=t(1, 3, 64, 128)), "multiple of heads_kv"),
])
def test_fused_fwd_rejects(bad, match):
    q, k, v = qkv()
    args = dict(q=q, k=k, v=v)
    kw = {}
    for name, val in bad.items():
        (args if name in args else kw)[name] = val
    with pytest.raises(ValueError, match=match):
        pb.fused_fwd(args["q"], args["k"], args["v"], **kw)


def test_decode_rejects():
    q, k, v = qkv(B=2, Hq=8, Hkv=2, Sq=1, Skv=1000)
    with pytest.raises(ValueError, match="v .* must have k's shape"):
        pb.splitkv_decode(q, k, t(2, 2, 999, 128))
    with pytest.raises(ValueError, match="lse must have shape"):
        pb.splitkv_decode(q, k, v, lse=torch.empty(2, 8, 1, device=M))
    with pytest.raises(ValueError, match="out .* must have q's shape"):
        pb.splitkv_decode(q, k, v, out=t(2, 8, 1, 64))
    parts = pb.Parts.empty(3, 2, 8, 128, M)
    with pytest.raises(ValueError, match="parts must be"):
        pb.splitkv_decode(q, k, v, num_splits=4, parts=parts)


def test_combine_and_merge_reject():
    parts = pb.Parts.empty(3, 2, 8, 128, M)
    with pytest.raises(ValueError, match="out must be"):
        pb.combine(parts, out=t(2, 8, 2, 128))
    with pytest.raises(ValueError, match="lse must be"):
        pb.combine(parts, lse=torch.empty(2, 7, device=M))
    with pytest.raises(ValueError, match="acc must be"):
        pb.combine(parts, acc=pb.Parts.empty(2, 2, 8, 128, M), want_out=False)
    with pytest.raises(ValueError, match="lse_parts"):
        pb.merge_partials(t(3, 10, 128), torch.empty(3, 11, device=M))
    with pytest.raises(ValueError, match="out must be"):
        pb.merge_partials(t(3, 10, 128), torch.empty(3, 10, device=M), out=t(10, 64))
