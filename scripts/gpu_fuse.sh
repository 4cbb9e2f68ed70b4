cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py -k tcgen05 -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_engine.py -x -q -p no:cacheprovider 2>&1 | tail -2
for d in 0 2097152; do MOE_TC_DBG=$d timeout 300 python tools/tc_tps.py 0,128,256 64,256 | sed "s/^/dbg=$d /"; done
