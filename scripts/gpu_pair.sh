cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -k "tcgen05" -x -q -p no:cacheprovider 2>&1 | tail -4
for dbg in 0 16384 2048 6150; do MOE_TC_DBG=$dbg PREC=1 timeout 300 python tools/prefill_tf.py ${PTS:-1024,2048,4096} | sed "s/^/dbg=$dbg /"; done
