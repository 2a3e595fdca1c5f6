#!/usr/bin/env python
"""Run ONE hot-path launch configuration a few times for ncu (developer tool):
  profile_target.py prefill <workload>     (bench.py WORKLOADS name, the bench launch configuration)
  profile_target.py decode <B>             (config 5: Hq=32 Hkv=8 KV 128K D=128, default splits)
  profile_target.py softmax                (65536 x 4096 bf16 rows)
Launches: 3 warm-up + 2 (profile with ncu -s 3 -c 1)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import datagen  # noqa: E402
import paper_2510_08726_b200 as pb  # noqa: E402
from datagen import device as dgd  # noqa: E402


def main():
    kind = sys.argv[1]
    if kind == "prefill":
        cid, B, Hq, Hkv, S, D, var = bench.WORKLOADS[sys.argv[2]]
        seed = datagen.config_seed(cid)
        q = dgd.tensor(seed, 1, (B, Hq, S, D))
        k = dgd.tensor(seed, 2, (B, Hkv, S, D))
        v = dgd.tensor(seed, 3, (B, Hkv, S, D))
        o = torch.empty_like(q)
        kw = dict(causal=var.get("causal", False), window=var.get("window", (-1, -1)), softcap=var.get("softcap", 0.0))
        if var.get("alibi"):
            kw["alibi_slopes"] = torch.tensor(datagen.alibi_slopes(Hq), device="cuda")
        fn = lambda: pb.fused_fwd(q, k, v, out=o, **kw)  # noqa: E731
    elif kind == "decode":
        B, Hq, Hkv, L, D = int(sys.argv[2]), 32, 8, 131072, 128
        seed = datagen.config_seed(5)
        q = dgd.tensor(seed, 1, (B, Hq, 1, D))
        k = dgd.tensor(seed, 2, (B, Hkv, L, D))
        v = dgd.tensor(seed, 3, (B, Hkv, L, D))
        o = torch.empty_like(q)
        ws = torch.zeros(pb.workspace_bytes(q, k), dtype=torch.uint8, device="cuda")
        fn = lambda: pb.splitkv_decode(q, k, v, causal=True, out=o, workspace=ws)  # noqa: E731
    elif kind == "softmax":
        x = dgd.tensor(datagen.config_seed(6), 1, (65536, 4096))
        y = torch.empty_like(x)
        fn = lambda: pb.softmax_rows(x, out=y)  # noqa: E731
    else:
        raise SystemExit(__doc__)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
