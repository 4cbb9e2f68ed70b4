cd $GRAFT_REPO_ROOT
# A/B: precision groups in the persistent tcgen05 kernel (MOE_TCP_W4)
for r in 1 2; do
for w in 0 1500 2500 4000; do
  MOE_B200_LIB=$PWD/build/ab/libmoe_w$w.so timeout 200 python tools/tc_tps.py 128 32,64,128,256 2>&1 | grep tok/s | sed "s/^/W4=$w /"
done
done
for w in 2500; do
  MOE_B200_LIB=$PWD/build/ab/libmoe_w$w.so timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1 | sed "s/^/W4=$w tests: /"
done
