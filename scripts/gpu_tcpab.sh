cd $GRAFT_REPO_ROOT
for lib in base ${LIBS}; do
  if [ $lib = base ]; then unset MOE_B200_LIB; else export MOE_B200_LIB=$PWD/build/ab/libmoe_$lib.so; fi
  timeout 300 python tools/tc_tps.py ${N4S:-0,128} ${TS:-64,256} 2>&1 | grep tok/s | sed "s/^/$lib /"
done
