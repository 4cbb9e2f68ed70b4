cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -k "tcgen05" -x -q -p no:cacheprovider 2>&1 | tail -2
for x in 0 16384; do
  MOE_TC_DBG=$x PREC=1 timeout 120 python tools/prefill_tf.py 1024,2048,4096 2>&1 | grep bf16 | sed "s/^/dbg=$x /"
done
MOE_TC_DBG=32768 PREC=1 timeout 120 python tools/prefill_tf.py 4096 > gpurun_out/wtrace_el.log 2>&1
