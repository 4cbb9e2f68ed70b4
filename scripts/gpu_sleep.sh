cd $GRAFT_REPO_ROOT
# A/B: finisher poll sleep (MOE_FIN_SLEEP ns)
for r in 1 2; do
for v in 128 32 512 2000; do
  MOE_B200_LIB=$PWD/build/ab/libmoe_s$v.so timeout 150 python tools/flow_tps.py 0,128,256 2>&1 | grep tok/s | sed "s/^/sleep=$v /"
done
done
