cd $GRAFT_REPO_ROOT
timeout 120 python tools/flow_tps.py 0,128,256 | sed "s/^/8k 7x2 /"
export MOE_B200_LIB=$PWD/build/ab/libmoe_4k.so
for c in 7x2 11x2 15x2; do MOE_FLOW_CFG=$c timeout 120 python tools/flow_tps.py 0,128,256 | sed "s/^/4k $c /"; done
MOE_FLOW_CFG=11x2 timeout 300 python -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider 2>&1 | tail -2
