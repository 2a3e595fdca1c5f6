#!/bin/bash
# Decode A/B (developer tool): parity of build/var_$1, then fused-combine latency and B=1/4 GB/s for every build/var_*.
cd "$GRAFT_REPO_ROOT"
ATTN_LIB_PATH=$PWD/build/var_${1:-comb}/libattn.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -x -k "decode or combine or dist" -p no:cacheprovider 2>&1 | tail -2
for lib in build/var_*/libattn.so; do echo "== $lib"; ATTN_LIB_PATH=$PWD/$lib timeout 300 python tools/probe_decode_latency.py 2>&1 | grep "cfg5"; ATTN_LIB_PATH=$PWD/$lib BS="1 4" timeout 300 python tools/decode_splits.py 2>&1 | grep -E "splits=(18|4) " ; done
