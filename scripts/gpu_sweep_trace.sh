# env sweep (kernel timing + bench) then launch timelines for the given trace env sets
bash scripts/gpu_envsweep.sh
for envs in ${TRACE_ENVS:-"MRAB_DUMMY=0"}; do
  echo "== $envs"; env $envs python scripts/trace_step.py 2>&1 | head -${TRACE_LINES:-12}
done > gpurun_out/trace.txt 2>&1
cat gpurun_out/trace.txt
