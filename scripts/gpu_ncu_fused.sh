# ncu --set full of the fused step kernels (flow with MOE_BAR_MODE, and step) at N4
cd $GRAFT_REPO_ROOT
N4=${N4:-256}
for v in "flow ${BM:-0}" "step 0"; do set -- $v
MOE_FUSED=$1 MOE_BAR_MODE=$2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_ -s 3 -c 1 \
  -o gpurun_out/prof_$1_n4_$N4 python tools/flow_tps.py $N4 > gpurun_out/ncu_$1.log 2>&1; echo "ncu $1 rc=$?"
python tools/ncu_summary.py gpurun_out/prof_$1_n4_$N4.ncu-rep > gpurun_out/ncu_$1_summary.txt 2>&1
head -60 gpurun_out/ncu_$1_summary.txt
done
