#!/bin/bash
# Quick interleaved A/B with short per-run timeouts (developer tool).
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/ab_${1:-x}.log; : > $OUT
for r in $(seq ${ROUNDS:-1}); do for lib in build/var_*/libattn.so; do for w in ${WORKLOADS:-mha}; do
  ATTN_LIB_PATH=$PWD/$lib timeout ${TMO:-120} python bench.py --steps ${STEPS:-20} --warmup 5 --no-e2e --no-decode --no-cpu --no-softmax --no-workloads --workload $w 2>&1 | \
    python -c "import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$r $lib $w', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'clk', d['clocks'].get('sm_mhz'))" >> $OUT
done; done; done
cat $OUT
