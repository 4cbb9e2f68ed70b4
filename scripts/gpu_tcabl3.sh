cd $GRAFT_REPO_ROOT
for dbg in ${DBGS:-0 1 7}; do
MOE_TC_DBG=$dbg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_ffn" --csv --log-file gpurun_out/tcabl_$dbg.csv python tools/run_tc.py 256 64 1 > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/tcabl_$dbg.csv')) if len(r)>10]
h=rows[0]; agg={}
for r in rows[1:]:
    g=r[h.index('Grid Size')]; a=agg.setdefault(g,[0,0]); a[0]+=1; a[1]+=float(r[h.index('Metric Value')].replace(',',''))
print('dbg $dbg', {g: round(t/c/1000,1) for g,(c,t) in agg.items()})
PY
done
