cd $GRAFT_REPO_ROOT
for r in 1 2; do
for v in cur fin; do
  MOE_B200_LIB=$PWD/build/ab/libmoe_$v.so timeout 150 python tools/flow_tps.py 0,128,256 2>&1 | grep tok/s | sed "s/^/$v /"
done
done

MOE_B200_LIB=$PWD/build/ab/libmoe_fin.so timeout 300 python -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider 2>&1 | tail -1 | sed "s/^/fin fused tests: /"
