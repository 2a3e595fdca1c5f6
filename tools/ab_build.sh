#!/bin/bash
# A/B builds of libattn.so (developer tool): build/var_<name>/libattn.so from a git revision
# ("name=rev") or from the working tree ("name=."), each with optional extra nvcc flags
# ("name=rev:-DFLAG").  Bench them with tools/gpu_variants.sh.
cd /root/repo
rm -rf build/var_*
for spec in "$@"; do
  n=${spec%%=*}; rest=${spec#*=}; rev=${rest%%:*}; flags=""; [[ "$rest" == *:* ]] && flags=${rest#*:}
  mkdir -p build/var_$n
  if [ "$rev" = "." ]; then src=/root/repo; else
    src=/tmp/ab_src_$n; rm -rf $src; mkdir -p $src
    git archive "$rev" paper_2510_08726_b200/csrc include | tar -x -C $src
  fi
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -diag-suppress 177 $flags -shared -o build/var_$n/libattn.so \
    $src/paper_2510_08726_b200/csrc/{api,fwd_tc,fwd_simt,decode,softmax_rows}.cu -ldl &
done
wait
ls build/var_*/libattn.so
