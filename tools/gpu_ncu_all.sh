#!/bin/bash
# ncu --set full of every benched kernel (one launch each) + the launch list of the default bench.
cd "$GRAFT_REPO_ROOT"
TAG=${1:-x}
mkdir -p gpurun_out/ncu_$TAG
for w in ${WORKLOADS:-mha mha_causal gqa_window var_scaled_dot var_alibi_causal var_softcap_causal}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_tc -s 3 -c 1 \
    -o gpurun_out/ncu_$TAG/fwd_$w python tools/profile_target.py prefill $w > /dev/null 2>&1
done
if [ -z "$NO_DECODE" ]; then
for b in 1 16; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_split -s 3 -c 1 \
    -o gpurun_out/ncu_$TAG/decode_b$b python tools/profile_target.py decode $b > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:softmax_rows -s 3 -c 1 \
  -o gpurun_out/ncu_$TAG/softmax_rows python tools/profile_target.py softmax > /dev/null 2>&1
fi
if [ -n "$LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
fi
ls -la gpurun_out/ncu_$TAG
# summarise on the box (the reports are too large to bring back all at once)
python tools/ncu_traffic.py gpurun_out/ncu_$TAG gpurun_out/ncu_full_summary_$TAG.json gpurun_out/ncu_traffic_$TAG.json > /dev/null
for f in gpurun_out/ncu_$TAG/*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  case " ${KEEP:-fwd_mha fwd_var_alibi_causal} " in *" $b "*) ;; *) rm -f $f ;; esac
done
