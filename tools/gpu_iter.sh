#!/bin/bash
# Fast iteration: prefill parity subset + prefill bench lines for every workload.
cd "$GRAFT_REPO_ROOT"
TAG=${1:-iter}
OUT=gpurun_out/iter_$TAG.log
: > $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "${PYTEST_K:-prefill or fp32}" --timeout 300 -p no:cacheprovider 2>&1 | tail -15 >> $OUT
for w in ${WORKLOADS:-mha mha_causal gqa_window var_scaled_dot var_alibi_causal var_softcap_causal}; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-decode --no-cpu --no-softmax --workload $w 2>&1 | \
    python -c "import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.rstrip()); continue
    print('$w', round(d['value'],1), 'TFLOP/s', 'frac', round(d['roofline']['frac'],3), 'ms', round(d['ms_per_step'],4), 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))" >> $OUT
done
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_tc -s 2 -c 1 -o gpurun_out/prof_fwd_$TAG \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-decode > /dev/null 2>&1
fi
cat $OUT
