"""Build build/libattn_trace.so (-DATTN_TRACE) and print a per-step timeline of one CTA of the MHA config."""
import ctypes, os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
lib_path = os.path.join(ROOT, "build", "libattn_trace%s.so" % os.environ.get("TRACE_TAG", ""))
if not os.path.exists(lib_path):
    src = [os.path.join(ROOT, "paper_2510_08726_b200", "csrc", f) for f in ("api.cu", "fwd_tc.cu", "fwd_simt.cu", "decode.cu", "softmax_rows.cu")]
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "-Xcompiler", "-fPIC", "-DATTN_TRACE", "-shared", "-o", lib_path] + os.environ.get("NVCC_EXTRA", "").split() + src)
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
tr = np.zeros((32, 16), dtype=np.int64)
ctypes.CDLL(lib_path).attn_debug_trace(tr.ctypes.data_as(ctypes.c_void_p))
t0 = tr[3, 0]
names = {24: "ld:K issue", 25: "ld:V issue", 12: "mma:V ready", 13: "mma:P0 seen", 15: "mma:K+1 ready", 14: "mma:P1 seen", 0: "mma:PV0 iss", 1: "mma:QK0+1 iss", 2: "mma:PV1 iss", 4: "sm0:wait S", 5: "sm0:S ready",
         6: "sm0:exp start", 7: "sm0:P done", 8: "sm1:wait S", 9: "sm1:S ready", 10: "sm1:exp start", 11: "sm1:P done", 16: "q0 exp end", 17: "q1 exp end", 18: "q2 exp end", 19: "q3 exp end", 20: "q1:S ready", 21: "q1:S regs", 22: "q1:max", 23: "q1:exp start", 26: "sm0:S regs", 27: "sm0:max", 28: "sm0:o_done", 29: "sm1:S regs", 30: "sm1:max", 31: "sm1:o_done"}
print("step " + " ".join(f"{names[e]:>13s}" for e in names))
for j in range(min(16, S // 128 + 1)):
    print(f"{j:4d} " + " ".join(f"{((tr[e, j] - t0) & 0xffffffff) if tr[e, j] else 0:13d}" for e in names))
# sorted event timeline of a few steady-state steps
print()
evs = []
for j in range(8, 11):
    for e, nm in names.items():
        if tr[e, j]:
            evs.append((int((tr[e, j] - t0) & 0xffffffff), j, nm))
evs.sort()
base = evs[0][0]
prev = base
for t, j, nm in evs:
    print(f"{t - base:7d} (+{t - prev:5d})  step {j:2d}  {nm}")
    prev = t
