# decode bench at n4 = 0 / 128 / 256 (3 rounds) + GPU tests
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2 3; do
for n4 in 0 128 256; do
  MOE_GEMV_DBG=${DBG:-0} timeout 600 python bench.py --n4 $n4 --steps 200 --warmup 5 --no-sweep --no-batch-sweep --no-prefill --no-host-split --no-reconfig --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n4=$n4', d['value'], d['roofline']['frac'])"
done
done
