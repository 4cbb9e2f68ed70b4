# round-2 re-entry check: smoke, full gpu tests, quick bench with sweep endpoints, fused phase trace
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --sweep-points 0,128,256 --no-cpu-baseline > gpurun_out/bench_quick.json 2>gpurun_out/bench_quick.err; echo "bench rc=$?"
python - <<'PY'
import json
l=json.loads(open('gpurun_out/bench_quick.json').read().strip().splitlines()[-1])
print('value', l['value'], 'roofline', l['roofline']['achieved'], l['roofline']['frac'], 'e2e', l['e2e']['value'])
for s in l['sweep']: print(s)
for s in l.get('batch_sweep', []): print(s)
for s in l.get('prefill_tcgen05', {}).get('points', []): print(s)
PY
for n in 256 128; do timeout 300 python tools/trace_fused.py $n; done > gpurun_out/trace_fused.txt 2>&1; cat gpurun_out/trace_fused.txt | tail -60
