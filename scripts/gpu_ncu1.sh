# one ncu --set full capture of the GEMV passes at N4 (default 256)
cd $GRAFT_REPO_ROOT
N4=${N4:-256}
TAG=${TAG:-x}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 130 -c 2 \
  -o gpurun_out/prof_${TAG}_n4_$N4 python bench.py --n4 $N4 --steps 2 --warmup 3 --no-sweep --no-cpu-baseline \
  > gpurun_out/ncu_${TAG}_$N4.log 2>&1; echo "ncu rc=$?"
