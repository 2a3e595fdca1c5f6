"""Small invocations of every kernel family, for compute-sanitizer runs (memcheck, racecheck,
synccheck): tcgen05 prefill (D=128 causal GQA -> persistent kernel; D=128 non-causal and ALiBi ->
grid kernel; D=64 plain / causal / softcap / ALiBi+window -> 64-key-tile kernel), KV-split prefill
(fp32 partials + merge), context-parallel partial, fp32 SIMT forward, split-KV decode (fused
combine, raw parts + combine, packed triples), softmax rows."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import datagen
import paper_2510_08726_b200 as pb
from datagen import device as dgd

q = dgd.tensor(1, 1, (1, 2, 300, 128)); k = dgd.tensor(1, 2, (1, 1, 300, 128)); v = dgd.tensor(1, 3, (1, 1, 300, 128))
sl2 = torch.tensor(datagen.alibi_slopes(2), device="cuda")
pb.fused_fwd(q, k, v, causal=True)
pb.fused_fwd(q, k, v)
pb.fused_fwd(q, k, v, causal=True, alibi_slopes=sl2)
q6, k6, v6 = (t[:, :, :, :64].contiguous() for t in (q, k, v))
pb.fused_fwd(q6, k6, v6)
pb.fused_fwd(q6, k6, v6, causal=True)
pb.fused_fwd(q6, k6, v6, causal=True, softcap=8.0)
pb.fused_fwd(q6, k6, v6, alibi_slopes=sl2, window=(100, 0))
ql = dgd.tensor(4, 1, (1, 2, 40, 128)); kl = dgd.tensor(4, 2, (1, 2, 2000, 128)); vl = dgd.tensor(4, 3, (1, 2, 2000, 128))
pb.fused_fwd(ql, kl, vl, causal=True, kv_splits=4)
pb.fused_fwd_partial(ql, kl, vl, kv_pos_offset=0, seqlen_kv_total=2000)
qf = dgd.tensor(1, 1, (1, 1, 64, 16), torch.float32)
pb.fused_fwd(qf, qf.clone(), qf.clone())
qd = dgd.tensor(2, 1, (1, 8, 1, 128)); kd = dgd.tensor(2, 2, (1, 2, 1000, 128)); vd = dgd.tensor(2, 3, (1, 2, 1000, 128))
pb.splitkv_decode(qd, kd, vd, num_splits=5, causal=True)
pb.splitkv_decode(qd, kd, vd, num_splits=5, causal=True, parts=pb.Parts.empty(5, 1, 8, 128, "cuda"))
pb.splitkv_decode(qd, kd, vd, num_splits=5, causal=True, packed=torch.empty(1, 8, 130, device="cuda"))
x = dgd.tensor(3, 1, (33, 1000))
pb.softmax_rows(x)
torch.cuda.synchronize()
print("sanitize workload done")
