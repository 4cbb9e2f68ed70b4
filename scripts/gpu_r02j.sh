# round-2 pass at HEAD (r02j: sentinel row hand-off): smoke, gpu tests, bench (+ reference arm), traffic, launch list, flow ncu, trace, tc tok/s
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --profile-from-start off --clock-control none \
  --csv --log-file gpurun_out/traffic.csv python tools/traffic.py run > gpurun_out/traffic_run.log 2>&1; echo "traffic rc=$?"
python tools/traffic.py summarize gpurun_out/traffic.csv gpurun_out/traffic_alg.json "$(cat build/commit.txt 2>/dev/null)" > profiles/r02_traffic.json; cat profiles/r02_traffic.json | head -30
cp profiles/r02_traffic.json gpurun_out/r02_traffic.json
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-600
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_|route|stream_kernel|finalize|tc_ffn|gather|combine" -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-batch-sweep --no-prefill --no-host-split --no-reconfig --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_ -s 3 -c 1 -o gpurun_out/prof_flow_n4_128_j python tools/flow_tps.py 128 > gpurun_out/ncu_flow.log 2>&1; echo "ncu flow rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_ -s 3 -c 1 -o gpurun_out/prof_flow_n4_256_j python tools/flow_tps.py 256 > gpurun_out/ncu_flow256.log 2>&1; echo "ncu flow 256 rc=$?"
for n in 256 128 0; do timeout 120 python tools/trace_fused.py $n; done > gpurun_out/trace_flow.txt 2>&1
timeout 200 python tools/tc_tps.py 0,128,256 64,256 > gpurun_out/tc_tps.txt 2>&1; cat gpurun_out/tc_tps.txt
