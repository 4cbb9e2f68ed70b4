cd $GRAFT_REPO_ROOT
N4=${N4:-256}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv -s 130 -c 2 -o gpurun_out/prof_gemv_$N4 python bench.py --n4 $N4 --steps 2 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/ncu_gemv.log 2>&1; echo "ncu rc=$?"
python bench.py --n4 $N4 --steps 50 --no-sweep --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300
