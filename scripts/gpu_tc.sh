# tcgen05 FFN: parity at 128- and 256-token tiles, then prefill / batch numbers
cd $GRAFT_REPO_ROOT
for dbg in 0 8 16; do
  echo "### MOE_TC_DBG=$dbg"
  MOE_TC_DBG=$dbg timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -p no:cacheprovider -k "tc or tcgen05" 2>&1 | tail -2
done
for dbg in 8 0; do
  MOE_TC_DBG=$dbg timeout 900 python bench.py --steps 20 --warmup 3 --no-sweep --no-host-split --no-reconfig --no-cpu-baseline --batch-points 64,128,256 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('dbg=$dbg batch', [(r['batch'], r['tokens_per_s']) for r in d['batch_sweep']])
print('dbg=$dbg prefill', [(p['tokens'], p['experts'], p['tflops']) for p in d['prefill_tcgen05']['points']])"
done
