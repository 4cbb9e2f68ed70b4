cd $GRAFT_REPO_ROOT
# A/B: sentinel x rows (HEAD lib in-tree) vs the counter hand-off (build/ab/libmoe_cur.so)
timeout 300 python -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider 2>&1 | tail -2 | sed "s/^/xs fused tests: /"
for r in 1 2; do
for v in cur xs; do
  if [ $v = xs ]; then L=; else L=$PWD/build/ab/libmoe_$v.so; fi
  MOE_B200_LIB=$L timeout 150 python tools/flow_tps.py 0,128,256 2>&1 | grep -v Warn | tail -3 | sed "s/^/$v /"
done
done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2 | sed "s/^/all gpu tests: /"
