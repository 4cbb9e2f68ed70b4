cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_kernels.py tests/test_gpu_stack.py tests/test_gpu_fused.py -x -q -p no:cacheprovider 2>&1 | tail -2
for d in 0 4194304; do MOE_TC_DBG=$d timeout 300 python tools/tc_tps.py 0,128 64,256 | sed "s/^/dbg=$d /"; done
