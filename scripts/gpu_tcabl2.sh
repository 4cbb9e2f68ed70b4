# tcgen05 ablation at batch-decode sizes (MOE_TC_DBG: bit0 skip convert, bit1 skip MMA, bit2 skip weight loads)
cd $GRAFT_REPO_ROOT
for dbg in 0 1 2 4 7; do
  MOE_TC_DBG=$dbg timeout 600 python bench.py --n4 ${N4:-128} --steps 10 --warmup 3 --no-sweep --no-prefill --no-host-split --no-reconfig --no-cpu-baseline --batch-points 64,256 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('dbg=$dbg', [(r['batch'], r['ms_per_step']) for r in d['batch_sweep']])"
done
