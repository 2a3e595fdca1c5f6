import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2510_08726_b200 as pb
def t(fn, n=50):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): fn()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g): fn()
    for _ in range(5): g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): g.replay()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3
Hq, Hkv, D = 64, 8, 128
for L, ns in [(64, 1), (1024, 1), (1024, 16), (8192, 1), (8192, 18), (32768, 18)]:
    q = torch.randn(1, Hq, 1, D, device="cuda", dtype=torch.float16)
    k = torch.randn(1, Hkv, L, D, device="cuda", dtype=torch.float16); v = torch.randn_like(k)
    o = torch.empty_like(q)
    ws = torch.zeros(pb.workspace_bytes(q, k, ns), dtype=torch.uint8, device="cuda")
    us = t(lambda: pb.splitkv_decode(q, k, v, num_splits=ns, out=o, workspace=ws))
    x = torch.empty(1, device="cuda")
    us0 = t(lambda: x.add_(1))
    print(f"L={L} splits={ns} decode_us={us:.1f} empty_kernel_us={us0:.1f}", flush=True)

# fused Eq. 8 combine vs raw partials only (no combine): config 5 shape at B = 1
Hq, Hkv, D = 32, 8, 128
for L, ns in [(64, 1), (64, 18), (131072, 18)]:
    q = torch.randn(1, Hq, 1, D, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(1, Hkv, L, D, device="cuda", dtype=torch.bfloat16); v = torch.randn_like(k)
    o = torch.empty_like(q)
    ws = torch.zeros(pb.workspace_bytes(q, k, ns), dtype=torch.uint8, device="cuda")
    parts = pb.Parts.empty(ns, 1, Hq, D, "cuda")
    us_f = t(lambda: pb.splitkv_decode(q, k, v, num_splits=ns, out=o, workspace=ws))
    us_p = t(lambda: pb.splitkv_decode(q, k, v, num_splits=ns, parts=parts, want_out=False, workspace=ws))
    print(f"cfg5 L={L} splits={ns} fused_us={us_f:.1f} partials_only_us={us_p:.1f}", flush=True)
