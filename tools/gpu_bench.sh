#!/bin/bash
# bench + ncu launch list + full captures of the two hot kernels (one GPU).
cd "$GRAFT_REPO_ROOT"
TAG=${1:-r1}
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_tc -s 2 -c 1 -o gpurun_out/prof_fwd_$TAG \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-decode > gpurun_out/ncu_fwd_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_split -s 2 -c 1 -o gpurun_out/prof_dec_$TAG \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_dec_$TAG.log 2>&1
ls -la gpurun_out
