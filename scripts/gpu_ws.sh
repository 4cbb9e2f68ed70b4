cd $GRAFT_REPO_ROOT
MOE_FLOW_CFG=ws timeout 300 python -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider 2>&1 | tail -2
for c in ws 7x2; do MOE_FLOW_CFG=$c timeout 120 python tools/flow_tps.py 0,128,256 | sed "s/^/$c /"; done
MOE_FLOW_CFG=ws timeout 120 python tools/trace_fused.py 256
