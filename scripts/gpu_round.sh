# full GPU pass: smoke, gpu tests, default bench, ncu launch list + full captures
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-400
Q="--no-sweep --no-batch-sweep --no-prefill --no-host-split --no-reconfig --no-cpu-baseline"
K='regex:route|stream_kernel|finalize|permute_rows|tc_ffn|to_f16|combine|residual'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 330 -c 330 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 $Q > gpurun_out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 130 -c 2 \
  -o gpurun_out/prof_stream_n4_128 python bench.py --steps 2 --warmup 3 $Q > gpurun_out/ncu_stream.log 2>&1; echo "ncu stream rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_ffn -s 4 -c 2 \
  -o gpurun_out/prof_tc_T256 python bench.py --tokens 256 --steps 2 --warmup 3 $Q > gpurun_out/ncu_tc.log 2>&1; echo "ncu tc rc=$?"
ls -la gpurun_out
