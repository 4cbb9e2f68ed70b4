cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -k tcgen05 -x -q -p no:cacheprovider 2>&1 | tail -1
LIBS="head" N4S=0,128,256 bash scripts/gpu_tcpab.sh
