cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py -k tcgen05 -x -q -p no:cacheprovider 2>&1 | tail -1
for r in 1 2; do for l in cur head; do if [ $l = head ]; then export MOE_B200_LIB=$PWD/build/ab/libmoe_head.so; else unset MOE_B200_LIB; fi; timeout 120 python tools/prefill_tf.py 2048,4096 | sed "s/^/$l /"; done; done
