# per-mesh k_rhs2d timing vs the y-streaming strip length (config 3)
rm -f gpurun_out/strip.txt
for s in 0 auto 2 4 8 16; do
  if [ "$s" = 0 ]; then export MRAB_STREAM=0; unset MRAB_STREAM_STRIP
  elif [ "$s" = auto ]; then export MRAB_STREAM=1; unset MRAB_STREAM_STRIP
  else export MRAB_STREAM=1; export MRAB_STREAM_STRIP=$s; fi
  python - <<'PY' >> gpurun_out/strip.txt 2>&1
import os, sys
sys.path.insert(0, os.getcwd())
import synth
from paper_1805_06607_b200 import mrab
p = synth.make_config(int(os.environ.get("CFG", "3")), "full")
plan = mrab.Plan(p); ctx = mrab.Context(plan, p.q0)
ctx.step(p.history_m - 1 + 3)
res = [ctx.time_kernel(0, g, reps=20, flush_l2=True) for g in range(len(p.meshes))]
print("strip", os.environ.get("MRAB_STREAM"), os.environ.get("MRAB_STREAM_STRIP"), [f"mesh{g}: {ms*1e3:.1f} us {by/ms/1e6:.0f} GB/s" for g, (ms, by) in enumerate(res)])
PY
done
export MRAB_STREAM=1; unset MRAB_STREAM_STRIP
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "rhs_parity or state_parity" > gpurun_out/strip_pytest.log 2>&1
tail -1 gpurun_out/strip_pytest.log
python bench.py --steps 100 --warmup 5 --no-cpu --no-srab > gpurun_out/strip_bench.json 2>/dev/null
python scripts/show_bench.py gpurun_out/strip_bench.json
cat gpurun_out/strip.txt
