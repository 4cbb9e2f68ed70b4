cd $GRAFT_REPO_ROOT
Q="--no-sweep --no-batch-sweep --no-prefill --no-host-split --no-reconfig --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_ffn -s 4 -c 2 \
  -o gpurun_out/prof_tc_${TAG:-v2} python bench.py --tokens 256 --steps 2 --warmup 3 $Q > gpurun_out/ncu_tc.log 2>&1; echo "ncu tc rc=$?"
