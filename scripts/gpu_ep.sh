# expert-parallel checks on one GPU: virtual-rank kernel test + the EP bench path over NCCL with 1 rank
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_ep.py -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py --ep --steps 10 --no-cpu-baseline --no-sweep --no-batch-sweep --no-prefill > gpurun_out/ep.log 2>&1; tail -25 gpurun_out/ep.log | cut -c1-600
