cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py -k tcgen05 -x -q -p no:cacheprovider 2>&1 | tail -3
for d in 0 8388608; do MOE_TC_DBG=$d timeout 120 python tools/prefill_tf.py 1024,2048,4096 | sed "s/^/dbg=$d /"; done
