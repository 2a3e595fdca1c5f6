"""Developer A/B for attn_softmax_rows: GB/s (x read + y write) per library build.
Usage: python tools/softmax_bench.py [lib.so ...]   (default: the in-tree build)"""
import json
import os
import subprocess
import sys

CHILD = r'''
import json, sys, torch
import paper_2510_08726_b200 as pb
res = {}
for dt, rows, cols in [("bf16", 65536, 4096), ("bf16", 262144, 1024), ("bf16", 32768, 8192),
                       ("bf16", 16384, 16384), ("bf16", 8192, 32768), ("f16", 65536, 4096), ("f32", 65536, 4096)]:
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}[dt]
    x = torch.randn(rows, cols, device="cuda").mul_(3).to(tdt)
    y = torch.empty_like(x)
    for _ in range(5):
        pb.softmax_rows(x, out=y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 30
    a.record()
    for _ in range(n):
        pb.softmax_rows(x, out=y)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    res[f"{dt}_{rows}x{cols}"] = round(2 * x.numel() * x.element_size() / ms / 1e6, 1)
print(json.dumps(res))
'''

libs = sys.argv[1:] or [""]
for lib in libs:
    env = dict(os.environ)
    if lib:
        env["ATTN_LIB_PATH"] = os.path.abspath(lib)
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
    print(lib or "in-tree", out.stdout.strip() or out.stderr.strip()[-500:], flush=True)
