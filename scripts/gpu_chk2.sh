cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 120 python tools/prefill_tf.py 2048,4096
