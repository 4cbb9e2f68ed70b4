# ncu evidence: launch list of one decode step + full captures of the GEMV
# (int4-only plan and bf16-only plan).  Usage: bash scripts/gpu_prof.sh
cd $GRAFT_REPO_ROOT
K='regex:gemv|route|permute_rows|combine|gate|moe_'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 640 -c 256 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline \
  > gpurun_out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
for N4 in ${N4S:-256 0}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv -s 130 -c 2 \
  -o gpurun_out/prof_gemv_n4_$N4 python bench.py --n4 $N4 --steps 2 --warmup 3 --no-sweep --no-cpu-baseline \
  > gpurun_out/ncu_full_$N4.log 2>&1; echo "ncu full n4=$N4 rc=$?"
done
ls -la gpurun_out
