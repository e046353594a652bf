# per-mesh k_rhs2d timing for tile variants (config ${CFG:-3})
for v in ${VARIANTS:-0 3}; do
  MRAB_K2D=$v python - <<'PY' >> gpurun_out/sweep.txt 2>&1
import os, sys
sys.path.insert(0, os.getcwd())
import synth
from paper_1805_06607_b200 import mrab
p = synth.make_config(int(os.environ.get("CFG", "3")), "full")
plan = mrab.Plan(p); ctx = mrab.Context(plan, p.q0)
ctx.step(p.history_m - 1 + 3)
res = [ctx.time_kernel(0, g, reps=20, flush_l2=True) for g in range(len(p.meshes))]
print("variant", os.environ["MRAB_K2D"], [f"mesh{g}: {ms*1e3:.1f} us {by/ms/1e6:.0f} GB/s" for g, (ms, by) in enumerate(res)])
PY
  MRAB_K2D=$v python bench.py --steps 100 --warmup 5 --no-cpu --no-srab > gpurun_out/sweep_$v.json 2>/dev/null
  MRAB_K2D=$v MRAB_OVERLAP=0 python bench.py --steps 100 --warmup 5 --no-cpu --no-srab > gpurun_out/sweep_noov_$v.json 2>/dev/null
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "rhs_parity or state_parity" > gpurun_out/sweep_pytest.log 2>&1
tail -1 gpurun_out/sweep_pytest.log
cat gpurun_out/sweep.txt
