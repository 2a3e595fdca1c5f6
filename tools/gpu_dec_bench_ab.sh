cd "$GRAFT_REPO_ROOT"
for r in 1 2; do for lib in build/var_*/libattn.so; do
  ATTN_LIB_PATH=$PWD/$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu --no-softmax --no-workloads --workload mha 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); sw=d['decode']['batch_sweep']
print('$r $lib', {b: round(v['GB/s']) for b,v in sw.items()})"
done; done
