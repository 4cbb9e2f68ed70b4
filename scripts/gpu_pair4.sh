cd $GRAFT_REPO_ROOT
for r in 1 2 3; do for dbg in 0 1048576 262144; do MOE_TC_DBG=$dbg PREC=1 timeout 120 python tools/prefill_tf.py 2048,4096 2>&1 | sed "s/^/dbg=$dbg /"; done; done
