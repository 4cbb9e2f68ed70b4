# per-warp and per-kernel timelines of one Mixtral layer (int4 and bf16, T=1)
cd $GRAFT_REPO_ROOT
for p in 0 1; do
  timeout 300 python tools/trace_gemv.py $p 1 2>&1 | tail -16
  timeout 300 python tools/trace_layer.py $p 1 2>&1 | tail -12
done
