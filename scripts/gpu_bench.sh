# smoke + GPU tests + default bench + reference arm + traffic capture + launch list
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider ${K:+-k "$K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --profile-from-start off \
  --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/traffic.py run > gpurun_out/traffic.log 2>&1; echo "traffic rc=$?"
python tools/traffic.py summarize gpurun_out/traffic.csv gpurun_out/traffic_alg.json > gpurun_out/r02_traffic.json; cp gpurun_out/r02_traffic.json profiles/ 2>/dev/null
timeout 1500 python bench.py --steps ${STEPS:-20} --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps ${STEPS:-20} --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -c 400 gpurun_out/bench_ref.json
