# launch timelines of the config-3 macro step, default and split schedules
for envs in ${TRACE_ENVS:-"MRAB_OVERLAP=0" "MRAB_OVERLAP=1"}; do
  echo "== $envs"; env $envs python scripts/trace_step.py
done > gpurun_out/trace.txt 2>&1
cat gpurun_out/trace.txt
