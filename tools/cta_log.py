"""Per-CTA lifetimes of one prefill launch (trace build): duration stats, SM occupancy gaps, waves.
   python tools/cta_log.py [causal]   (TRACE_CFG=B,H,S,D, TRACE_TAG as trace_fwd.py)"""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
lib_path = os.path.join(ROOT, "build", "libattn_trace%s.so" % os.environ.get("TRACE_TAG", ""))
import torch
from paper_2510_08726_b200 import _ffi
_ffi.load(lib_path)
import paper_2510_08726_b200 as pb
from datagen import device as dgd
B, H, S, D = (int(x) for x in os.environ.get("TRACE_CFG", "8,16,4096,128").split(","))
q, k, v = (dgd.tensor(1, i, (B, H, S, D)) for i in (1, 2, 3))
causal = len(sys.argv) > 1 and sys.argv[1] == "causal"
for _ in range(3):
    o = pb.fused_fwd(q, k, v, causal=causal)
torch.cuda.synchronize()
lg = np.zeros((8192, 4), dtype=np.uint64)
ctypes.CDLL(lib_path).attn_debug_cta_log(lg.ctypes.data_as(ctypes.c_void_p))
n = int((lg[:, 1] > 0).sum())
lg = lg[:n].astype(np.int64)
t0 = lg[:, 0].min()
st, en, sm = lg[:, 0] - t0, lg[:, 1] - t0, lg[:, 2]
dur = en - st
cyc = lg[:, 3]
print(f"SM clock over CTA lifetimes: {np.median(cyc / dur):.3f} GHz; CTA cycles mean {cyc.mean():.0f}")
print(f"CTAs {n}, kernel span {en.max() / 1e3:.1f} us, CTA duration mean {dur.mean() / 1e3:.2f} us "
      f"min {dur.min() / 1e3:.2f} max {dur.max() / 1e3:.2f} p10 {np.percentile(dur, 10) / 1e3:.2f} p90 {np.percentile(dur, 90) / 1e3:.2f}")
busy = np.zeros(sm.max() + 1)
gaps = []
for s_ in range(sm.max() + 1):
    idx = np.where(sm == s_)[0]
    if len(idx) == 0:
        continue
    o_ = idx[np.argsort(st[idx])]
    busy[s_] = dur[o_].sum()
    gaps += list(st[o_][1:] - en[o_][:-1])
print(f"SM busy fraction mean {busy.mean() / en.max():.3f} (min {busy[busy > 0].min() / en.max():.3f}); "
      f"gap between CTAs on an SM: mean {np.mean(gaps) / 1e3:.2f} us, max {np.max(gaps) / 1e3:.2f} us; "
      f"last CTA start {st.max() / 1e3:.1f} us")
for w in range(0, n, 148):
    d = dur[w:w + 148]
    print(f"  CTAs {w:5d}..: start {st[w:w+148].min() / 1e3:7.1f}-{st[w:w+148].max() / 1e3:7.1f} us  dur mean {d.mean() / 1e3:6.2f} us")
