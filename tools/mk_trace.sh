#!/bin/bash
# usage: mk_trace.sh name [extra nvcc flags]
n=$1; shift
cd /root/repo
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DATTN_TRACE "$@" -shared -o build/libattn_trace_$n.so paper_2510_08726_b200/csrc/{api,fwd_tc,fwd_simt,decode,softmax_rows}.cu -ldl 2>&1 | grep -E " error"
ls -la build/libattn_trace_$n.so
