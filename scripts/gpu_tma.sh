timeout 300 python scripts/one_rhs_launch.py > gpurun_out/one.log 2>&1; tail -2 gpurun_out/one.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "rhs_parity or state_parity or config3 or full3" > gpurun_out/pytest_iter.log 2>&1
tail -3 gpurun_out/pytest_iter.log
rm -f gpurun_out/sweep.txt; VARIANTS=0 bash scripts/k2d_sweep.sh > /dev/null 2>&1; cat gpurun_out/sweep.txt
MRAB_TMA=0 python bench.py --steps 100 --warmup 5 --no-cpu --no-srab > gpurun_out/bench_notma.json 2>/dev/null
python bench.py --steps 100 --warmup 5 > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err
tail -2 gpurun_out/bench_iter.err
