"""Developer probe: per-CTA fixed cost of the prefill kernel.  Shapes with exactly 16 waves of
CTAs (2368 = 16 x 148) and 16..128 KV steps per CTA; fits time/wave = steps * period + overhead."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2510_08726_b200 as pb

rows = []
for S, H in ((2048, 296), (4096, 148), (8192, 74), (16384, 37)):
    q = torch.randn(1, H, S, 128, device="cuda", dtype=torch.bfloat16)
    k, v = torch.randn_like(q), torch.randn_like(q)
    for _ in range(3):
        pb.fused_fwd(q, k, v)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        pb.fused_fwd(q, k, v)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    steps = S // 128
    tf = 4 * 128 * S * S * H / ms / 1e9
    rows.append((steps, ms * 1e3 / 16))
    print(f"S={S} H={H} steps/CTA={steps} ms={ms:.4f} TFLOP/s={tf:.1f} us/wave={ms * 1e3 / 16:.2f}", flush=True)
x = np.array([r[0] for r in rows], float)
y = np.array([r[1] for r in rows], float)
p, o = np.polyfit(x, y, 1)
print(f"fit: period {p:.4f} us/step ({p * 1965:.0f} cycles at 1965 MHz), overhead {o:.2f} us/CTA ({o * 1965:.0f} cycles)")
