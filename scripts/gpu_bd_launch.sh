cd $GRAFT_REPO_ROOT
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bd_launches.csv python tools/tc_tps.py ${N4:-0} 256 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/bd_launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
seq=[(r[ki].split('(')[0][-40:], float(r[vi].replace(',',''))/1000) for r in rows[1:]]
# one step = the last 32 layers' worth: find per-kernel totals over the last N launches of one decode
per=collections.defaultdict(lambda:[0,0.0])
last=seq[-int(len(seq)/ (16+3+1+1)):]  # rough: last step
for n,us in last: per[n][0]+=1; per[n][1]+=us
tot=sum(v[1] for v in per.values())
print('launches in window', len(last), 'total us', round(tot,1))
for n,(c,us) in sorted(per.items(), key=lambda x:-x[1][1]): print(f'{us:9.1f} us {c:4d}x  {n}')
PY
