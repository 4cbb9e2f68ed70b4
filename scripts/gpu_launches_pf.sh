cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -k "tcgen05" -x -q -p no:cacheprovider 2>&1 | tail -2
PREC=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pf_launches.csv python tools/prefill_tf.py 4096 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/pf_launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
seq=[(r[ki][:60], float(r[vi].replace(',',''))/1000) for r in rows[1:]]
for name,us in seq[-12:]: print(f'{us:9.1f} us  {name}')
PY
