"""Small invocations of every kernel family, for compute-sanitizer runs."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import datagen
import paper_2510_08726_b200 as pb
from datagen import device as dgd

q = dgd.tensor(1, 1, (1, 2, 300, 128)); k = dgd.tensor(1, 2, (1, 1, 300, 128)); v = dgd.tensor(1, 3, (1, 1, 300, 128))
pb.fused_fwd(q, k, v, causal=True)
pb.fused_fwd(q[:, :, :, :64].contiguous(), k[:, :, :, :64].contiguous(), v[:, :, :, :64].contiguous(),
             alibi_slopes=torch.tensor(datagen.alibi_slopes(2), device="cuda"), window=(100, 0))
qf = dgd.tensor(1, 1, (1, 1, 64, 16), torch.float32)
pb.fused_fwd(qf, qf.clone(), qf.clone())
qd = dgd.tensor(2, 1, (1, 8, 1, 128)); kd = dgd.tensor(2, 2, (1, 2, 1000, 128)); vd = dgd.tensor(2, 3, (1, 2, 1000, 128))
pb.splitkv_decode(qd, kd, vd, num_splits=5, causal=True)
x = dgd.tensor(3, 1, (33, 1000))
pb.softmax_rows(x)
torch.cuda.synchronize()
print("sanitize workload done")
