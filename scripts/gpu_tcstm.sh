cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -k "tcgen05" -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_numerics.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 200 python tools/tc_tps.py 0,128,256 64,256
timeout 300 python tools/prefill_tf.py 512,2048,4096
