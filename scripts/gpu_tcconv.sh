cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -k "tcgen05" -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 300 python -m pytest tests/test_gpu_numerics.py -x -q -p no:cacheprovider 2>&1 | tail -2
DBGS="0 64" bash scripts/gpu_tcabl3.sh
timeout 200 python tools/tc_tps.py 0,128,256 64,256
