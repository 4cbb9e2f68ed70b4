cd $GRAFT_REPO_ROOT
for m in 0 1 2 3; do MOE_BAR_MODE=$m timeout 120 python tools/flow_tps.py 128,256; done 2>&1 | grep -v Warn
MOE_FUSED=step timeout 120 python tools/flow_tps.py 128,256
