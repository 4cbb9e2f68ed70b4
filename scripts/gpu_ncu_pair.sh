cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/pf.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import bench, paper_2407_14417_b200 as moe
prof1 = moe.profile_for_shape(bench.D_MODEL, bench.D_FFN, 1, bench.EXPERTS, bench.TOPK)
plan1 = moe.assign_locations([1] * bench.EXPERTS, moe.HardwareProfile(10**15), prof1)
eng = moe.MoeEngine(1, bench.EXPERTS, bench.TOPK, bench.D_MODEL, bench.D_FFN, plan1, max_tokens=4096, seed=0, norm_eps=bench.NORM_EPS)
eng.synth_input(1, 4096)
for _ in range(3):
    eng.decode(4096)
eng.sync()
PY
for dbg in 0 16384; do
MOE_TC_DBG=$dbg timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_ffn -s 2 -c 2 \
  -o gpurun_out/prof_pair_$dbg python /tmp/pf.py > gpurun_out/ncu_pair_$dbg.log 2>&1; echo "ncu $dbg rc=$?"
done
