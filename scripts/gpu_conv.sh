cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py -k "tcgen05" -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 300 python tools/tc_tps.py 0,128,256 64,256
MOE_TC_DBG=32768 timeout 120 python tools/run_tc.py 256 256 1 > gpurun_out/ptrace.log 2>&1
PREC=0 timeout 120 python tools/prefill_tf.py 2048,4096
