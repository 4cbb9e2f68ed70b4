cd $GRAFT_REPO_ROOT
for f in tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_ep.py tests/test_capi.py; do
  timeout 150 python -m pytest $f -m gpu -v -x -p no:cacheprovider > gpurun_out/t_$(basename $f).log 2>&1; echo "$f rc=$?"; tail -3 gpurun_out/t_$(basename $f).log
done
