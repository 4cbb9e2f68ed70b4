set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
nproc; free -g; ulimit -l; lscpu | grep -E "Model name|Socket|Thread|Core"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-sweep --no-cpu-baseline > gpurun_out/bench1.log 2>&1; echo bench rc=$?
tail -5 gpurun_out/bench1.log
