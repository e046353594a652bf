# march kernel: parity (forced), kernel timings, bench, trace map
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "march" > gpurun_out/pytest_march.log 2>&1; echo "rc $?" >> gpurun_out/pytest_march.log
tail -3 gpurun_out/pytest_march.log
for envs in ${TIMES:-"MRAB_MARCH=1"}; do
  env $envs REPS=10 python scripts/one_rhs_launch.py 2>&1 | tail -1 | sed "s/^/$envs /"
done
MARCH_MAP=1 python scripts/trace_step.py 2>&1 | head -${TRACE_LINES:-70} > gpurun_out/trace.txt; cat gpurun_out/trace.txt
