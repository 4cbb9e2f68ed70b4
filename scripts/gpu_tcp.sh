cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -k "tcgen05" -x -q -p no:cacheprovider 2>&1 | tail -3
DBGS="0 512 256" bash scripts/gpu_tcabl3.sh
for dbg in 0 512; do MOE_TC_DBG=$dbg timeout 200 python tools/tc_tps.py 0,128,256 64,256 | sed "s/^/dbg=$dbg /"; done
