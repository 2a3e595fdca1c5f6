"""Developer probe: decode GB/s vs split count (config 5, B = 1 and 4), CUDA-graph replay."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_08726_b200 as pb

Hq, Hkv, L, D = (int(os.environ.get(k, d)) for k, d in (("HQ", 32), ("HKV", 8), ("L", 131072), ("D", 128)))
for B in [int(x) for x in os.environ.get("BS", "1 2 4 8 16").split()]:
    q = torch.randn(B, Hq, 1, D, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(B, Hkv, L, D, device="cuda", dtype=torch.bfloat16)
    v = torch.randn_like(k)
    o = torch.empty_like(q)
    base = pb.default_splits(q, k)
    units = B * Hkv
    cands = {base, max(1, 148 // units), max(1, 148 // units) + 1, max(1, 296 // units), max(1, 444 // units),
             max(1, 1184 // units), max(1, 140 // units)}
    for ns in sorted(cands):
        if ns < 1:
            continue
        ws = torch.zeros(pb.workspace_bytes(q, k, ns), dtype=torch.uint8, device="cuda")
        step = lambda: pb.splitkv_decode(q, k, v, num_splits=ns, out=o, workspace=ws)  # noqa: E731
        step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step()
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            step()
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 50
        print(f"B={B} splits={ns} ctas={ns * B * Hkv} us={ms * 1e3:.1f} GB/s={2 * B * Hkv * L * D * 2 / ms / 1e6:.0f}", flush=True)
