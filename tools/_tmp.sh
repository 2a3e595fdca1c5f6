cd $GRAFT_REPO_ROOT
ATTN_LIB_PATH=$PWD/build/var_f2on/libattn.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
WORKLOADS="mha mha_causal gqa_window var_scaled_dot var_alibi_causal var_softcap_causal" timeout 900 bash tools/gpu_variants.sh f2
