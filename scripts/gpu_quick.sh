cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py --steps 100 --sweep-points ${SWEEP:-0,128,256} --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench_quick.json 2>gpurun_out/bench_quick.err
python - <<'PY'
import json
l=json.loads(open('gpurun_out/bench_quick.json').read().strip().splitlines()[-1])
print('value', l['value'], 'roofline', l['roofline']['achieved'], l['roofline']['frac'], 'e2e', l['e2e']['value'])
for s in l['sweep']: print(s)
for s in l.get('batch_sweep', []): print(s)
for s in l.get('prefill_tcgen05', {}).get('points', []): print(s)
PY
