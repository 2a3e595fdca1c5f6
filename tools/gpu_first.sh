#!/bin/bash
# First GPU bring-up: each test group in its own process (a trapped kernel poisons the CUDA context).
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
for grp in "test_device_generator or fp32" "decode or combine" "prefill_small" "rectangular or strided or host" "full_config"; do
  echo "=== $grp" >> gpurun_out/pytest1.log
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$grp" --timeout 300 -p no:cacheprovider 2>&1 | tail -40 >> gpurun_out/pytest1.log
done
