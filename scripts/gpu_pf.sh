# k_rhs2d timing vs the L2 prefetch mode MRAB_PF (config ${CFG:-3}), then parity + bench
rm -f gpurun_out/pf.txt
for pf in ${PFS:-0 1}; do
  MRAB_PF=$pf python - <<'PY' >> gpurun_out/pf.txt 2>&1
import os, sys
sys.path.insert(0, os.getcwd())
import synth
from paper_1805_06607_b200 import mrab
p = synth.make_config(int(os.environ.get("CFG", "3")), "full")
plan = mrab.Plan(p); ctx = mrab.Context(plan, p.q0)
ctx.step(p.history_m - 1 + 3)
res = [ctx.time_kernel(0, g, reps=20, flush_l2=True) for g in range(len(p.meshes))]
print("pf", os.environ["MRAB_PF"], [f"mesh{g}: {ms*1e3:.1f} us {by/ms/1e6:.0f} GB/s" for g, (ms, by) in enumerate(res)])
PY
  MRAB_PF=$pf python bench.py --steps 100 --warmup 5 --no-cpu --no-srab > gpurun_out/pf_bench_$pf.json 2>/dev/null
  python scripts/show_bench.py gpurun_out/pf_bench_$pf.json | head -2 >> gpurun_out/pf.txt
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "rhs_parity or state_parity" > gpurun_out/pf_pytest.log 2>&1
tail -1 gpurun_out/pf_pytest.log
cat gpurun_out/pf.txt
