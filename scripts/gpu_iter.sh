# quick iteration on the GPU box: 3-D parity tests, then short config-4 / config-5 bench lines
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout ${PT_TIMEOUT:-900} python -m pytest tests/test_gpu_parity.py -x -q ${PT_K:+-k "$PT_K"} > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_iter.log
tail -15 gpurun_out/pytest_iter.log
for c in ${BENCH_CFGS:-4}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu --no-srab --no-secondary > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  python scripts/show_bench.py gpurun_out/bench_c$c.json 2>/dev/null || tail -5 gpurun_out/bench_c$c.err
done
