cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 600 python bench.py --steps 200 --warmup 5 --no-sweep --no-batch-sweep --no-host-split --no-reconfig --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('headline', d['value'], d['roofline']['frac'])
print('prefill', [(p['tokens'], p['experts'], p['tflops']) for p in d['prefill_tcgen05']['points']])"
timeout 600 python bench.py --n4 0 --steps 100 --warmup 5 --no-sweep --no-prefill --no-host-split --no-reconfig --no-cpu-baseline --batch-points 1,8,64,256 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('n4=0', d['value'], d['roofline']['frac'], [(r['batch'], r['tokens_per_s']) for r in d['batch_sweep']])"
