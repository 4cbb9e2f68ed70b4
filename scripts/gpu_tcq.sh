cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -k "tcgen05" -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 300 python tools/tc_tps.py ${N4S:-0,128,256} ${TS:-64,256}
PREC=0 timeout 120 python tools/prefill_tf.py 2048,4096
