cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_fused.py -x -q -p no:cacheprovider 2>&1 | tail -2
for dbg in 0 262144; do MOE_TC_DBG=$dbg timeout 120 python tools/prefill_tf.py 512,1024,2048,4096 2>&1 | sed "s/^/dbg=$dbg /"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_ffn -s 0 -c 2 -o gpurun_out/prof_tc_wide2_4096 python tools/prefill_tf.py 4096 > gpurun_out/ncu_w2.log 2>&1; echo "ncu rc=$?"
