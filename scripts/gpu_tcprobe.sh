cd $GRAFT_REPO_ROOT
for n4 in 0 256; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"tc_ffn|gather|route|combine|permute" --csv --log-file gpurun_out/tc_launch_$n4.csv python tools/run_tc.py $n4 64 1 > /dev/null 2>&1; echo "rc=$?"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ffn -s 2 -c 2 -o gpurun_out/prof_tc64_n4_0 python tools/run_tc.py 0 64 1 > /dev/null 2>&1; echo "full rc=$?"
timeout 200 python tools/tc_tps.py 0,256 64,256
