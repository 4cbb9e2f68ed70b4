cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_kernels.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 300 python tools/tc_tps.py 0,128,256 64,256
export MOE_B200_LIB=$PWD/build/ab/libmoe_prev.so; timeout 300 python tools/tc_tps.py 0,128 64,256 | sed "s/^/prev /"
