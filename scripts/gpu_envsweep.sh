# k_rhs timing + bench line per environment setting; SWEEP="A=1 B=2;A=0" (';'-separated), then parity
rm -f gpurun_out/envsweep.txt
IFS=';' read -ra SETS <<< "${SWEEP:-MRAB_DUMMY=0}"
i=0
for envs in "${SETS[@]}"; do
  i=$((i+1))
  echo "== $envs" >> gpurun_out/envsweep.txt
  env $envs python - <<'PY' >> gpurun_out/envsweep.txt 2>&1
import os, sys
sys.path.insert(0, os.getcwd())
import synth
from paper_1805_06607_b200 import mrab
p = synth.make_config(int(os.environ.get("CFG", "3")), "full")
plan = mrab.Plan(p); ctx = mrab.Context(plan, p.q0)
ctx.step(p.history_m - 1 + 3)
res = [ctx.time_kernel(0, g, reps=20, flush_l2=True) for g in range(len(p.meshes))]
print([f"mesh{g}: {ms*1e3:.1f} us {by/ms/1e6:.0f} GB/s" for g, (ms, by) in enumerate(res)])
PY
  env $envs python bench.py --config ${CFG:-3} --steps 100 --warmup 5 --no-cpu --no-srab > gpurun_out/envsweep_$i.json 2>/dev/null
  python scripts/show_bench.py gpurun_out/envsweep_$i.json 2>/dev/null | head -2 >> gpurun_out/envsweep.txt
done
if [ -n "$PARITY" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "$PARITY" > gpurun_out/envsweep_pytest.log 2>&1
  tail -1 gpurun_out/envsweep_pytest.log >> gpurun_out/envsweep.txt
fi
cat gpurun_out/envsweep.txt
