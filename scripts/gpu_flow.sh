# dataflow fused step: parity tests, phase trace, A/B vs the grid-barrier step and per-layer kernels
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider > gpurun_out/pytest_fused.log 2>&1; echo "fused tests rc=$?"; tail -15 gpurun_out/pytest_fused.log
for n in ${N4S:-256 128}; do timeout 120 python tools/trace_fused.py $n; done > gpurun_out/trace_flow.txt 2>&1; cat gpurun_out/trace_flow.txt
timeout 400 python tools/ab_fused.py ${AB:-0,128,256} > gpurun_out/ab_fused.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/ab_fused.txt
