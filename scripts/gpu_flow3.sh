cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 120 python tools/flow_tps.py 0,128,256
for n in 256 128; do timeout 120 python tools/trace_fused.py $n; done 2>&1
