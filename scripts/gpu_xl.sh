cd $GRAFT_REPO_ROOT
for r in 1 2; do
for v in xl dg4 dg2; do
  if [ $v = none ]; then L=; else L=$PWD/build/ab/libmoe_$v.so; fi
  MOE_B200_LIB=$L timeout 150 python tools/flow_tps.py 0,128,256 2>&1 | grep tok/s | sed "s/^/$v /"
done
done

