# round evidence: GPU tests, smoke, default bench line, launch list and ncu capture of the
# dominant kernels (each ncu pass only after its own command exited 0 without ncu)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_default_20.json 2> gpurun_out/bench_default_20.err
for c in ${EXTRA_CFGS:-}; do timeout 900 python bench.py --config $c --no-cpu > gpurun_out/bench_config$c.json 2> gpurun_out/bench_config$c.err; done
if [ -n "$NCU" ]; then
  python bench.py --steps 3 --warmup 3 --no-srab --no-cpu --no-secondary > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-srab --no-cpu --no-secondary > gpurun_out/ncu_launch.log 2>&1
  OUT=dominant bash scripts/gpu_ncu3d.sh
fi
CFG=4 timeout 300 python scripts/trace_step3d.py > gpurun_out/trace3d_c4_serial.txt 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -1; cat gpurun_out/bench_default.json
