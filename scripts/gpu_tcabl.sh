# tcgen05 ablation at prefill sizes (MOE_TC_DBG: bit0 skip convert, bit1 skip MMA, bit2 skip weight loads)
cd $GRAFT_REPO_ROOT
for dbg in ${DBGS:-0 1 2 4}; do
  MOE_TC_DBG=$dbg timeout 600 python bench.py --steps 5 --warmup 3 --no-sweep --no-batch-sweep --no-host-split --no-reconfig --no-cpu-baseline --prefill-points 4096 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('dbg=$dbg', [(p['experts'], p['ffn_ms'], p['tflops']) for p in d['prefill_tcgen05']['points']])"
done
