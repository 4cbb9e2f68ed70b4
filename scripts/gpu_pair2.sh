cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py -k "tcgen05" -x -q -p no:cacheprovider 2>&1 | tail -1
for lib in base ${LIBS}; do
  if [ $lib = base ]; then unset MOE_B200_LIB; else export MOE_B200_LIB=$PWD/build/ab/libmoe_$lib.so; fi
  PREC=1 timeout 120 python tools/prefill_tf.py 2048,4096 2>&1 | grep bf16 | sed "s/^/$lib /"
done
unset MOE_B200_LIB
MOE_TC_DBG=32768 PREC=1 timeout 120 python tools/prefill_tf.py 4096 > gpurun_out/w2trace.log 2>&1
