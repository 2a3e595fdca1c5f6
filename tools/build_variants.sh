#!/bin/bash
# Build A/B variants of libattn.so into build/var_<name>/ (developer tool).
# Usage: build_variants.sh name="-DFLAG ..." [name2="..."]
cd /root/repo
rm -rf build/var_*
for spec in "$@"; do
  n=${spec%%=*}; flags=${spec#*=}
  mkdir -p build/var_$n
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -diag-suppress 177 $flags -shared \
    -o build/var_$n/libattn.so paper_2510_08726_b200/csrc/{api,fwd_tc,fwd_simt,decode,softmax_rows}.cu &
done
wait
ls build/var_*/libattn.so
