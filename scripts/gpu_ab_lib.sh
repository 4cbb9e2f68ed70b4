# A/B of an alternative library build (build/ab/$LIBAB) against the in-tree one
cd $GRAFT_REPO_ROOT
timeout 120 python tools/flow_tps.py ${PTS:-0,128,256}
MOE_B200_LIB=$PWD/build/ab/$LIBAB timeout 120 python tools/flow_tps.py ${PTS:-0,128,256}
MOE_B200_LIB=$PWD/build/ab/$LIBAB timeout 300 python -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider 2>&1 | tail -2
