"""NEXT-4 workload: the paper's Fig. 2 reduction chain (attn_softmax_rows) on
the GPU against oracle.softmax_rows (fp64), for every dtype, single-chunk and
multi-chunk rows, ragged tails, masked (-inf) entries, empty rows and strides."""
import numpy as np
import pytest
import torch

import datagen
import oracle
from datagen import device as dgd
from tests.helpers import assert_bf16_close

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2510_08726_b200 as pb


def _inputs(rows, cols, dtype, seed, stride=None):
    x32 = datagen.tensor(seed, 1, (rows, cols), "f32") * np.float32(3.0)
    x32[1 % rows, ::5] = -np.inf                   # masked entries
    if rows > 3:
        x32[3, :] = -np.inf                          # an empty row
    if dtype == "bf16":
        bits = datagen.f32_to_bf16_bits(x32)
        x64 = datagen.as_f64(bits, "bf16")
    elif dtype == "f16":
        bits = x32.astype(np.float16).view(np.uint16)
        x64 = datagen.as_f64(bits, "f16")
    else:
        bits, x64 = x32, x32.astype(np.float64)
    t = dgd.to_device(np.ascontiguousarray(bits), dtype=dtype)
    if stride is not None:
        big = torch.zeros(rows, stride, dtype=t.dtype, device="cuda")
        big[:, :cols] = t
        t = big[:, :cols]
    return t, x64


@pytest.mark.parametrize("dtype", ["bf16", "f16", "f32"])
@pytest.mark.parametrize("cols", [1, 7, 100, 1000, 4096, 8192, 8200, 20000])
def test_softmax_rows(dtype, cols):
    rows = 9
    x, x64 = _inputs(rows, cols, dtype, seed=cols, stride=cols + 24 if cols % 8 == 0 else None)
    if cols % 8:      # contiguous rows need a 16-byte-multiple stride: pad
        x, x64 = _inputs(rows, cols, dtype, seed=cols, stride=((cols + 7) // 8) * 8)
    y, m, l = pb.softmax_rows(x, return_stats=True)
    rm, rl, ry = oracle.softmax_rows(x64)
    yg = y.float().cpu().numpy().astype(np.float64)
    if dtype == "f32":
        assert np.abs(yg - ry).max() <= 1e-4
    else:
        assert_bf16_close(yg, ry, f"softmax rows {dtype} cols={cols}")
    mg, lg = m.cpu().numpy(), l.cpu().numpy()
    fin = np.isfinite(rm)
    assert np.array_equal(np.isfinite(mg), fin)
    np.testing.assert_allclose(mg[fin], rm[fin], rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(lg, rl, rtol=1e-4, atol=1e-30)
    assert np.all(yg[~fin] == 0)


def test_softmax_rows_stats_only_large():
    """Fig. 2a's outputs alone (row max, row sum) on a BASELINE-scale block of rows."""
    rows, cols = 512, 4096
    x, x64 = _inputs(rows, cols, "bf16", seed=3)
    _, m, l = pb.softmax_rows(x, want_out=False, return_stats=True)
    rm, rl, _ = oracle.softmax_rows(x64)
    fin = np.isfinite(rm)
    np.testing.assert_allclose(m.cpu().numpy()[fin], rm[fin], rtol=1e-6)
    np.testing.assert_allclose(l.cpu().numpy(), rl, rtol=1e-4)
