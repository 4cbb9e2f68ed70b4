# honest per-pass ncu of the per-layer streaming GEMV (int4 gate/up and down, n4=256) and the fused step
cd $GRAFT_REPO_ROOT
cat > /tmp/run_pl.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import paper_2407_14417_b200 as moe
prof = moe.profile_for_shape(4096, 14336, 32, 8, 2)
plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, 256, 0), moe.HardwareProfile(10**15), prof)
eng = moe.MoeEngine(32, 8, 2, 4096, 14336, plan, max_tokens=1, seed=0, norm_eps=1e-5, use_graphs=False, per_layer_decode=True)
eng.synth_input(7, 1)
for _ in range(2):
    eng.decode(1)
eng.sync()
print("ok")
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 64 -c 2 -o gpurun_out/prof_stream_n4_256 python /tmp/run_pl.py > gpurun_out/ncu_stream.log 2>&1; echo "ncu stream rc=$?"
