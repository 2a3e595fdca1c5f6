#!/bin/bash
# Interleaved A/B of build/var_*/libattn.so: ROUNDS x (each variant x each workload), one line per run.
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/ab_${1:-x}.log; : > $OUT
for r in $(seq ${ROUNDS:-2}); do
  for lib in build/var_*/libattn.so; do
    for w in ${WORKLOADS:-mha mha_causal}; do
      ATTN_LIB_PATH=$PWD/$lib timeout 300 python bench.py --steps ${STEPS:-20} --warmup 5 --no-e2e --no-decode --no-cpu --no-softmax --workload $w 2>&1 | \
        python -c "import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.rstrip()[:300]); continue
    print('$r $lib $w', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'clk', d['clocks'].get('sm_mhz'))" >> $OUT
    done
  done
done
cat $OUT
