#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over tools/sanitize.py: production build,
# then synccheck on the ATTN_STRICT_WAITS build (build/libattn_strict.so) and a GPU parity run of
# the strict build (its o_done assertions trap if the skipped-phase invariant were ever violated).
cd "$GRAFT_REPO_ROOT"
TAG=${1:-x}
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize.py > gpurun_out/sanitize_${tool}_$TAG.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_${tool}_$TAG.log
  tail -3 gpurun_out/sanitize_${tool}_$TAG.log
done
ATTN_LIB_PATH=$PWD/build/libattn_strict.so timeout 900 compute-sanitizer --tool synccheck python tools/sanitize.py \
  > gpurun_out/sanitize_synccheck_strict_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize_synccheck_strict_$TAG.log
tail -3 gpurun_out/sanitize_synccheck_strict_$TAG.log
ATTN_LIB_PATH=$PWD/build/libattn_strict.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_repair.py \
  -m gpu -q --timeout 300 -p no:cacheprovider -k "64" 2>&1 | tail -2
