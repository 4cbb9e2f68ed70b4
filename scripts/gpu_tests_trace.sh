# GPU tests (optional -k $K) + isolated-layer kernel timelines
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider ${K:+-k "$K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
for p in 0 1; do timeout 300 python tools/trace_layer.py $p 1 1; done > gpurun_out/trace_layer.txt 2>&1; cat gpurun_out/trace_layer.txt
