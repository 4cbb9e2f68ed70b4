# A/B of MOE_GEMV_DBG settings on the decode bench (n4 = 128 / 256), back to back, 2 rounds + int4/bf16 layer traces
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do
for n4 in 0 128 256; do
for dbg in ${DBGS:-0 64}; do
  MOE_GEMV_DBG=$dbg timeout 600 python bench.py --n4 $n4 --steps 200 --warmup 5 --no-sweep --no-batch-sweep --no-prefill --no-host-split --no-reconfig --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n4=$n4 dbg=$dbg', d['value'])"
done
done
done
for dbg in ${DBGS:-0 64}; do for p in 0 1; do MOE_GEMV_DBG=$dbg timeout 300 python tools/trace_layer.py $p 1 2>&1 | grep -E "gate/up|span"; done; done
