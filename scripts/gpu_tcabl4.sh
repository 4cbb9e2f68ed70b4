cd $GRAFT_REPO_ROOT
for dbg in 0 4096; do
MOE_TC_DBG=$dbg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_ffn" --csv --log-file gpurun_out/tcabl4_$dbg.csv python tools/run_tc.py 256 64 1 > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/tcabl4_$dbg.csv')) if len(r)>10]
h=rows[0]; v=[float(r[h.index('Metric Value')].replace(',','')) for r in rows[1:]]
print('dbg $dbg', 'gate/up avg', round(sum(v[0::2])/len(v[0::2])/1000,1), 'down avg', round(sum(v[1::2])/len(v[1::2])/1000,1))
PY
done
