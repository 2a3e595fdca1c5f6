#!/bin/bash
# Round checkpoint: full GPU test suite, smoke, bench (all keys), launch list, ncu captures.
cd "$GRAFT_REPO_ROOT"
TAG=${1:-ck}
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
for w in mha_causal gqa_window var_scaled_dot var_alibi_causal var_softcap_causal var_causal var_alibi mha_alibi mha_alibi_causal; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-decode --no-cpu --no-softmax --workload $w >> gpurun_out/bench_workloads_$TAG.jsonl 2>/dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
if [ -n "$NCU_FULL" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_tc -s 2 -c 1 -o gpurun_out/prof_fwd_$TAG \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-decode > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_split -s 2 -c 1 -o gpurun_out/prof_dec_$TAG \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:softmax_rows -s 2 -c 1 -o gpurun_out/prof_smr_$TAG \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-decode > /dev/null 2>&1
fi
if [ -n "$SANITIZE" ]; then
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool python tools/sanitize.py > gpurun_out/sanitize_${tool}_$TAG.log 2>&1
    echo "rc=$?" >> gpurun_out/sanitize_${tool}_$TAG.log
  done
fi
tail -3 gpurun_out/pytest_$TAG.log
