#!/bin/bash
# Full checkpoint + the Table 3 grid (tag as $1).
cd "$GRAFT_REPO_ROOT"
TAG=${1:-ck}
NCU_FULL=1 SANITIZE=1 bash tools/gpu_full.sh $TAG
timeout 600 python tools/sweep.py --table3 --dtype fp16 > gpurun_out/table3_$TAG.json 2> gpurun_out/table3_$TAG.err
timeout 600 python tools/decode_splits.py > gpurun_out/decode_splits_$TAG.txt 2>&1
