cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -k "tcgen05" -x -q -p no:cacheprovider 2>&1 | tail -2
for dbg in 0 128; do MOE_TC_DBG=$dbg timeout 300 python tools/prefill_tf.py ${PTS:-2048,4096} | sed "s/^/dbg=$dbg /"; done
