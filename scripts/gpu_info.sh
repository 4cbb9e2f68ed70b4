# box info + smoke + GPU tests (baseline state at the start of a round)
cd $GRAFT_REPO_ROOT
{ free -g; nproc; lscpu | grep -E "Model name|Socket|Thread|NUMA node\(s\)"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; } > gpurun_out/boxinfo.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
