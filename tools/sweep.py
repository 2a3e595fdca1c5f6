#!/usr/bin/env python
"""The paper's operator sweep on B200, our kernels only (NEXT-1).

Table 1: ten LLM attention operators, prefill (PF: s_q = s_kv) and
decode (DC: s_q = 1), seq 2^7..2^15, batch 1, fp16.  The paper
names only the base architectures; the head shapes below are those models'
published attention shapes (reading R14 in DESIGN.md).  Timing follows the
paper's protocol: warm-up, then the mean of timed runs (CUDA
events, no L2 flush).  Also the batch-scalability curve (GQA PF, seq 8192,
P:1191-1213).  Writes one JSON document to stdout.

  python tools/sweep.py [--dtype fp16|bf16] [--reps 15] [--max-log2 15]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2510_08726_b200 as pb  # noqa: E402
from datagen import device as dgd  # noqa: E402

# name: (mode, base arch, Hq, Hkv, D, variant)
OPERATORS = {
    "Global (PF)": ("PF", "ViT-L/16", 16, 16, 64, dict()),
    "Causal (PF)": ("PF", "GPT-3 6.7B", 32, 32, 128, dict(causal=True)),
    "GQA (PF)": ("PF", "Llama-3 70B", 64, 8, 128, dict(causal=True)),
    "ALiBi (PF)": ("PF", "MPT-7B", 32, 32, 128, dict(causal=True, alibi=True)),
    "SoftCap (PF)": ("PF", "Gemma-2 27B", 32, 16, 128, dict(causal=True, softcap=50.0)),
    "Window (PF)": ("PF", "(window 4096, Mistral-7B shape)", 32, 8, 128, dict(causal=True, window=(4095, 0))),
    "Causal (DC)": ("DC", "GPT-3 6.7B", 32, 32, 128, dict(causal=True)),
    "GQA (DC)": ("DC", "Llama-3 70B", 64, 8, 128, dict(causal=True)),
    "ALiBi (DC)": ("DC", "MPT-7B", 32, 32, 128, dict(causal=True, alibi=True)),
    "SoftCap (DC)": ("DC", "Gemma-2 27B", 32, 16, 128, dict(causal=True, softcap=50.0)),
}


def pairs(Sq, Skv, var):
    causal = var.get("causal", False)
    wl, wr = var.get("window", (-1, -1))
    off = Skv - Sq
    tot = 0
    for i in range(Sq):
        qp = off + i
        lo = max(0, qp - wl) if wl >= 0 else 0
        hi = Skv - 1
        if causal:
            hi = min(hi, qp)
        if wr >= 0:
            hi = min(hi, qp + wr)
        tot += max(0, hi - lo + 1)
    return tot


def time_fn(fn, reps, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(reps):
        fn()
    s1.record()
    torch.cuda.synchronize()
    return s0.elapsed_time(s1) / reps


def time_graph(fn, reps):
    """Same step captured in a CUDA graph and replayed: the GPU time without the
    Python binding's per-call host cost (which dominates launch-bound shapes)."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return time_fn(g.replay, reps)


def run_op(name, seq, B, dtype, reps):
    mode, arch, Hq, Hkv, D, var = OPERATORS[name]
    tdt = torch.float16 if dtype == "fp16" else torch.bfloat16
    Sq = seq if mode == "PF" else 1
    q = dgd.tensor(7, 1, (B, Hq, Sq, D), tdt)
    k = dgd.tensor(7, 2, (B, Hkv, seq, D), tdt)
    v = dgd.tensor(7, 3, (B, Hkv, seq, D), tdt)
    kw = dict(causal=var.get("causal", False), window=var.get("window", (-1, -1)), softcap=var.get("softcap", 0.0))
    if var.get("alibi"):
        kw["alibi_slopes"] = torch.tensor(datagen.alibi_slopes(Hq), device="cuda")
    out = torch.empty_like(q)
    if mode == "PF":
        fn = lambda: pb.fused_fwd(q, k, v, out=out, **kw)  # noqa: E731
    else:
        ws = torch.zeros(pb.workspace_bytes(q, k), dtype=torch.uint8, device="cuda")   # ticket block starts at 0
        fn = lambda: pb.splitkv_decode(q, k, v, out=out, workspace=ws, **kw)  # noqa: E731
    ms = time_fn(fn, reps)
    flops = 4.0 * D * pairs(Sq, seq, var) * B * Hq
    kv_bytes = 2.0 * B * Hkv * seq * D * 2
    return {"op": name, "mode": mode, "arch": arch, "B": B, "Hq": Hq, "Hkv": Hkv, "D": D, "seq": seq,
            "ms": ms, "TFLOP/s": flops / (ms * 1e-3) / 1e12, "KV GB/s": kv_bytes / (ms * 1e-3) / 1e9}


def run_table3(reps, dtype):
    """Table 3's grid: global (non-causal) attention, s_q <= s_kv,
    s_q in 16..2048, s_kv in 128..2048 (chunked prefill / multi-token shapes, NEXT-2).
    The paper gives no head shape for it: B = 1, 32 heads, D = 128 (reading R15)."""
    tdt = torch.float16 if dtype == "fp16" else torch.bfloat16
    out = []
    for skv in (128, 256, 512, 1024, 2048):
        for sq in (16, 32, 64, 128, 256, 512, 1024, 2048):
            if sq > skv:
                continue
            q = dgd.tensor(8, 1, (1, 32, sq, 128), tdt)
            k = dgd.tensor(8, 2, (1, 32, skv, 128), tdt)
            v = dgd.tensor(8, 3, (1, 32, skv, 128), tdt)
            o = torch.empty_like(q)
            fn = lambda: pb.fused_fwd(q, k, v, out=o)  # noqa: E731
            ms = time_fn(fn, reps)
            msg = time_graph(fn, reps)
            flops = 4.0 * 128 * sq * skv * 32
            out.append({"s_q": sq, "s_kv": skv, "us": ms * 1e3, "TFLOP/s": flops / (ms * 1e-3) / 1e12,
                        "us_graph": msg * 1e3, "TFLOP/s_graph": flops / (msg * 1e-3) / 1e12})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="fp16", choices=["fp16", "bf16"])
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--max-log2", type=int, default=15)
    ap.add_argument("--ops", default="all")
    ap.add_argument("--table3", action="store_true", help="only the s_q x s_kv grid of Table 3")
    args = ap.parse_args()
    if args.table3:
        print(json.dumps({"dtype": args.dtype, "table3": run_table3(args.reps, args.dtype)}, indent=1))
        return
    ops = list(OPERATORS) if args.ops == "all" else [o for o in OPERATORS if o.split()[0] in args.ops.split(",")]
    res = {"dtype": args.dtype, "protocol": f"mean of {args.reps} runs after 3 warm-ups, CUDA events, no L2 flush "
           "(the paper's protocol P:1006-1011)", "operators": [], "batch_scaling": []}
    for name in ops:
        for lg in range(7, args.max_log2 + 1):
            res["operators"].append(run_op(name, 2 ** lg, 1, args.dtype, args.reps))
            torch.cuda.empty_cache()
    for B in (1, 2, 4, 8, 16, 32):
        res["batch_scaling"].append(run_op("GQA (PF)", 8192, B, args.dtype, max(3, args.reps // 3)))
        torch.cuda.empty_cache()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
