# quick 3-D kernel iteration: 3-D parity, then config 4 / 5 bench lines
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "${PT_K:-rhs or state}" > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_iter.log
tail -4 gpurun_out/pytest_iter.log
for c in ${BENCH_CFGS:-4 5}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu --no-srab --no-secondary > gpurun_out/bench_c${c}.json 2> gpurun_out/bench_c${c}.err
  echo "config $c"; python scripts/show_bench.py gpurun_out/bench_c${c}.json 2>/dev/null || tail -5 gpurun_out/bench_c${c}.err
done
