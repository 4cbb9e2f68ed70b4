cd $GRAFT_REPO_ROOT
for lib in base cur; do
  if [ $lib = base ]; then export MOE_B200_LIB=$PWD/build/ab/libmoe_base.so; else unset MOE_B200_LIB; fi
  for n4 in 0 256; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_ffn" --csv --log-file gpurun_out/tcab_${lib}_${n4}.csv python tools/run_tc.py $n4 64 1 > /dev/null 2>&1
  python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/tcab_${lib}_${n4}.csv')) if len(r)>10]
h=rows[0]; agg={}
for r in rows[1:]:
    g=r[h.index('Grid Size')]; a=agg.setdefault(g,[0,0]); a[0]+=1; a[1]+=float(r[h.index('Metric Value')].replace(',',''))
print('$lib n4=$n4', {g: round(t/c/1000,1) for g,(c,t) in agg.items()})
PY
  done
done
