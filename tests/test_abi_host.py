"""C-ABI library: loads without a GPU, exports every symbol include/attn.h
declares, and rejects bad arguments with the documented status codes before
touching the device (argument checks are synchronous and host-only)."""
import ctypes
import os
import re

import pytest

from paper_2510_08726_b200 import _ffi
from paper_2510_08726_b200._ffi import AttnParts, AttnProblem, AttnTensor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_ffi.LIB_PATH):
        from paper_2510_08726_b200 import build
        build.build()
    return _ffi.load()


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "attn.h")).read()
    return sorted(set(re.findall(r"ATTN_API\s+[\w\s\*]+?\b(attn_\w+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    declared = _declared_symbols()
    assert len(declared) >= 9
    assert set(declared) == set(_ffi.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.attn_abi_version() == 1


def test_datagen_library_exports():
    path = os.path.join(ROOT, "datagen", "libdatagen.so")
    if not os.path.exists(path):
        from paper_2510_08726_b200 import build
        build.build()
    assert hasattr(ctypes.CDLL(path), "datagen_fill")


def _prob(**kw):
    p = AttnProblem(batch=1, heads_q=4, heads_kv=2, seqlen_q=16, seqlen_kv=16, head_dim=128, dtype=_ffi.ATTN_BF16,
                    scale=0.1, softcap=0.0, alibi_slopes=None, causal=0, window_left=-1, window_right=-1,
                    seqlen_kv_total=0, q_pos_offset=_ffi.ATTN_Q_POS_DEFAULT, kv_pos_offset=0)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


FAKE = 0x7F0000000000  # never dereferenced: every case below fails validation first


def _t(ptr=FAKE, sb=4 * 16 * 128, sh=16 * 128, ss=128):
    return AttnTensor(ptr, sb, sh, ss)


@pytest.mark.parametrize("kw,status", [
    (dict(heads_q=3), _ffi.ATTN_ERR_INVALID_ARGUMENT),
    (dict(seqlen_q=0), _ffi.ATTN_ERR_INVALID_ARGUMENT),
    (dict(scale=0.0), _ffi.ATTN_ERR_INVALID_ARGUMENT),
    (dict(scale=float("inf")), _ffi.ATTN_ERR_INVALID_ARGUMENT),
    (dict(softcap=-1.0), _ffi.ATTN_ERR_INVALID_ARGUMENT),
    (dict(window_left=-2), _ffi.ATTN_ERR_INVALID_ARGUMENT),
    (dict(kv_pos_offset=5, seqlen_kv_total=16), _ffi.ATTN_ERR_INVALID_ARGUMENT),
    (dict(head_dim=96), _ffi.ATTN_ERR_UNSUPPORTED),
    (dict(dtype=_ffi.ATTN_FP32, head_dim=512), _ffi.ATTN_ERR_UNSUPPORTED),
    (dict(dtype=7), _ffi.ATTN_ERR_INVALID_ARGUMENT),
])
def test_fused_fwd_argument_errors(lib, kw, status):
    p = _prob(**kw)
    st = lib.attn_fused_fwd(ctypes.byref(p), _t(), _t(), _t(), _t(), None, None)
    assert st == status, lib.attn_last_error()
    assert lib.attn_last_error()


def test_alignment_errors(lib):
    p = _prob()
    assert lib.attn_fused_fwd(ctypes.byref(p), _t(FAKE + 2), _t(), _t(), _t(), None, None) == _ffi.ATTN_ERR_ALIGNMENT
    assert lib.attn_fused_fwd(ctypes.byref(p), _t(ss=100), _t(), _t(), _t(), None, None) == _ffi.ATTN_ERR_ALIGNMENT
    assert lib.attn_fused_fwd(ctypes.byref(p), _t(0), _t(), _t(), _t(), None, None) == _ffi.ATTN_ERR_INVALID_ARGUMENT


def test_decode_errors(lib):
    p = _prob(seqlen_q=2)    # multi-token decode (G * Sq = 4 rows) is supported: here it needs workspace
    nul = AttnTensor(None, 0, 0, 0)
    st = lib.attn_splitkv_decode(ctypes.byref(p), _t(), _t(), _t(), 0, None, 0, None, _t(), None, None)
    assert st == _ffi.ATTN_ERR_WORKSPACE_TOO_SMALL
    p = _prob(seqlen_q=1)
    st = lib.attn_splitkv_decode(ctypes.byref(p), _t(), _t(), _t(), 0, None, 0, None, nul, None, None)
    assert st == _ffi.ATTN_ERR_INVALID_ARGUMENT          # neither parts nor o
    st = lib.attn_splitkv_decode(ctypes.byref(p), _t(), _t(), _t(), 4, None, 0, None, _t(), None, None)
    assert st == _ffi.ATTN_ERR_WORKSPACE_TOO_SMALL
    parts = AttnParts(FAKE, FAKE, FAKE, 3, 0, 0, 0, 0, 0, 0)
    st = lib.attn_splitkv_decode(ctypes.byref(p), _t(), _t(), _t(), 4, None, 0, ctypes.byref(parts), nul, None, None)
    assert st == _ffi.ATTN_ERR_INVALID_ARGUMENT          # num_parts != splits
    p = _prob(seqlen_q=1, heads_q=32, heads_kv=1)
    st = lib.attn_splitkv_decode(ctypes.byref(p), _t(), _t(), _t(), 0, None, 0, None, _t(), None, None)
    assert st == _ffi.ATTN_ERR_UNSUPPORTED              # group of 32 rows > one 16-row tile
    p = _prob(seqlen_q=5, heads_q=8, heads_kv=2)
    st = lib.attn_splitkv_decode(ctypes.byref(p), _t(), _t(), _t(), 0, None, 0, None, _t(), None, None)
    assert st == _ffi.ATTN_ERR_UNSUPPORTED              # G * seqlen_q = 20 > 16
    p = _prob(seqlen_q=2, heads_q=8, heads_kv=2)
    parts = AttnParts(FAKE, FAKE, FAKE, 1, 0, 0, 0, 0, 0, 0)
    st = lib.attn_splitkv_decode(ctypes.byref(p), _t(), _t(), _t(), 1, None, 0, ctypes.byref(parts), _t(), None, None)
    assert st == _ffi.ATTN_ERR_UNSUPPORTED              # raw triples only for seqlen_q == 1


def test_workspace_and_splits_are_host_functions(lib):
    p = _prob(seqlen_q=1, batch=1, heads_q=32, heads_kv=8, seqlen_kv=131072)
    s = lib.attn_splitkv_default_splits(ctypes.byref(p), 148)
    assert s == 148 // 8                                    # one CTA per SM, one wave
    ws = lib.attn_splitkv_workspace_bytes(ctypes.byref(p), s)
    assert ws >= s * 32 * (128 + 2) * 4
    p.seqlen_kv = 10
    assert lib.attn_splitkv_default_splits(ctypes.byref(p), 148) == 1


def test_combine_errors(lib):
    nul = AttnTensor(None, 0, 0, 0)
    parts = AttnParts(FAKE, FAKE, FAKE, 2, 0, 0, 0, 0, 0, 0)
    assert lib.attn_combine(1, 1, 128, ctypes.byref(parts), 0, nul, None, None, None) == _ffi.ATTN_ERR_INVALID_ARGUMENT
    assert lib.attn_combine(1, 1, 512, ctypes.byref(parts), 0, _t(), None, None, None) == _ffi.ATTN_ERR_UNSUPPORTED
    bad = AttnParts(FAKE, FAKE, FAKE, 2, 0, 0, 0, 0, 0, 0)
    assert lib.attn_combine(1, 1, 128, ctypes.byref(parts), 0, _t(), None, ctypes.byref(bad), None) == \
        _ffi.ATTN_ERR_INVALID_ARGUMENT


def test_status_strings(lib):
    for s in range(6):
        assert lib.attn_status_string(s)


def test_product_package_does_not_import_oracle():
    """The product path must never route through the oracle."""
    pkg = os.path.join(ROOT, "paper_2510_08726_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"\boracle\b", src.replace("oracle/", "")) or "import oracle" not in src, f
                assert "import oracle" not in src and "from oracle" not in src, f


def test_nccl_entry_points_host_side(lib):
    """The multi-GPU entry points: NCCL is dlopen'ed at run time (ncclGetUniqueId
    needs no GPU); argument errors come back as status codes."""
    buf = ctypes.create_string_buffer(128)
    assert lib.attn_nccl_get_unique_id(buf) == _ffi.ATTN_OK
    assert any(buf.raw)
    assert lib.attn_nccl_get_unique_id(None) == _ffi.ATTN_ERR_INVALID_ARGUMENT
    assert lib.attn_nccl_comm_destroy(None) == _ffi.ATTN_OK
    h = ctypes.c_void_p()
    assert lib.attn_nccl_comm_init(ctypes.byref(h), 2, 2, buf) == _ffi.ATTN_ERR_INVALID_ARGUMENT   # rank >= nranks
    p = _prob(seqlen_q=1, batch=2, heads_q=32, heads_kv=8, seqlen_kv=16384)
    ws = lib.attn_decode_kv_sharded_workspace_bytes(ctypes.byref(p), 8)
    assert ws >= (8 + 1) * 2 * 32 * 130 * 4                # send + nranks receive slots
    assert lib.attn_decode_kv_sharded(None, ctypes.byref(p), _t(), _t(), _t(), None, 0, _t(), None, None) == \
        _ffi.ATTN_ERR_INVALID_ARGUMENT


def test_prefill_split_heuristic_is_host_only(lib):
    """attn_fused_fwd_default_splits / _workspace_bytes (NEXT-2) are pure host functions."""
    big = _prob(batch=8, heads_q=16, heads_kv=16, seqlen_q=4096, seqlen_kv=4096)
    assert lib.attn_fused_fwd_default_splits(ctypes.byref(big), 148) == 1       # grid fills the GPU
    assert lib.attn_fused_fwd_workspace_bytes(ctypes.byref(big), 0) == 0
    small = _prob(batch=1, heads_q=32, heads_kv=32, seqlen_q=16, seqlen_kv=2048)
    assert lib.attn_fused_fwd_default_splits(ctypes.byref(small), 148) == 4     # 32 units -> 4 per unit
    ws = lib.attn_fused_fwd_workspace_bytes(ctypes.byref(small), 4)
    assert ws >= 4 * 32 * 16 * (128 * 2 + 4)
    short = _prob(batch=1, heads_q=2, heads_kv=2, seqlen_q=16, seqlen_kv=1024)
    assert lib.attn_fused_fwd_default_splits(ctypes.byref(short), 148) == 1     # 8 tiles: < 4 splits of 4
    wide = _prob(batch=1, heads_q=64, heads_kv=8, seqlen_q=512, seqlen_kv=8192)
    assert lib.attn_fused_fwd_default_splits(ctypes.byref(wide), 148) == 1      # 128 units: < 4 per unit
    f32 = _prob(batch=1, heads_q=2, heads_kv=2, seqlen_q=16, seqlen_kv=4096, dtype=_ffi.ATTN_FP32)
    assert lib.attn_fused_fwd_default_splits(ctypes.byref(f32), 148) == 1


def test_partial_and_packed_argument_errors(lib):
    """attn_fused_fwd_partial (fp32 CP partial) and attn_splitkv_decode_packed (the KV-sharded
    decode's send triple): host-side argument checks, no device access."""
    p = _prob()
    assert lib.attn_fused_fwd_partial(ctypes.byref(p), _t(), _t(), _t(), None, FAKE, None) == \
        _ffi.ATTN_ERR_INVALID_ARGUMENT                      # o_part required
    assert lib.attn_fused_fwd_partial(ctypes.byref(p), _t(), _t(), _t(), FAKE + 4, FAKE, None) == \
        _ffi.ATTN_ERR_ALIGNMENT                             # o_part 16-byte aligned
    f32 = _prob(dtype=_ffi.ATTN_FP32)
    assert lib.attn_fused_fwd_partial(ctypes.byref(f32), _t(), _t(), _t(), FAKE, FAKE, None) == \
        _ffi.ATTN_ERR_UNSUPPORTED                           # bf16 / fp16 inputs only
    d = _prob(seqlen_q=1)
    assert lib.attn_splitkv_decode_packed(ctypes.byref(d), _t(), _t(), _t(), 0, None, 0, None, None) == \
        _ffi.ATTN_ERR_INVALID_ARGUMENT                      # packed required
    assert lib.attn_splitkv_decode_packed(ctypes.byref(d), _t(), _t(), _t(), 0, None, 0, FAKE, None) == \
        _ffi.ATTN_ERR_WORKSPACE_TOO_SMALL                   # ticket workspace required
    m = _prob(seqlen_q=2)
    assert lib.attn_splitkv_decode_packed(ctypes.byref(m), _t(), _t(), _t(), 0, None, 0, FAKE, None) == \
        _ffi.ATTN_ERR_UNSUPPORTED                           # one query per (b, hq)


def test_repair_counter_hook_is_host_only(lib):
    """attn_debug_repair_counters only records a pointer (thread-local) for later calls."""
    lib.attn_debug_repair_counters(FAKE)
    lib.attn_debug_repair_counters(None)
