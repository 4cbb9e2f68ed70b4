cd $GRAFT_REPO_ROOT
for r in 1 2; do
for v in cur dup; do
  MOE_B200_LIB=$PWD/build/ab/libmoe_$v.so timeout 150 python tools/flow_tps.py 0,128,256 2>&1 | grep tok/s | sed "s/^/$v /"
done
done

