# expert-parallel bench on one box: --gpus N self-launches N ranks (sharing the
# box's GPUs); tiny shape first, then the Mixtral shape
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --gpus 2 --shape tiny --n4 8 --steps 10 --warmup 3 > gpurun_out/ep_tiny.log 2>&1; echo "ep tiny rc=$?"; tail -3 gpurun_out/ep_tiny.log | cut -c1-700
timeout 900 python bench.py --gpus ${EPN:-2} --steps 10 --warmup 3 > gpurun_out/ep.log 2>&1; echo "ep rc=$?"; tail -3 gpurun_out/ep.log | cut -c1-1500
