cd $GRAFT_REPO_ROOT
for lib in base ${LIBS}; do
  if [ $lib = base ]; then unset MOE_B200_LIB; else export MOE_B200_LIB=$PWD/build/ab/libmoe_$lib.so; fi
  PREC=1 timeout 120 python tools/prefill_tf.py ${PTS:-2048,4096} 2>&1 | grep bf16 | sed "s/^/$lib /"
done
