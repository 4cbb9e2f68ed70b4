# f3 on the GPU: new engine/pareto tests + the measured Mixtral sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py -q -p no:cacheprovider -k "host_streaming or pareto" 2>&1 | tail -3
timeout 1500 python tools/pareto_sweep.py --mem-range ${MEM:-24GB:96GB:24GB} --n4-grid ${GRID:-0,128,256} --steps ${STEPS:-8} \
    --out gpurun_out/pareto_mixtral.csv 2>&1 | tail -5
cat gpurun_out/pareto_mixtral.csv
