cd $GRAFT_REPO_ROOT
# A/B: breadth-first int4 groups in the dataflow step (MOE_FLOW_NG build knob)
for r in 1 2; do
for v in base ng2 ng4 ng8; do
  if [ $v = base ]; then L=; else L=$PWD/build/ab/libmoe_$v.so; fi
  MOE_B200_LIB=$L timeout 150 python tools/flow_tps.py 0,128,256 2>&1 | grep tok/s | sed "s/^/$v /"
done
done
for v in ng4 ng8; do
  MOE_B200_LIB=$PWD/build/ab/libmoe_$v.so timeout 300 python -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider 2>&1 | tail -1 | sed "s/^/$v fused tests: /"
done
