timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rhs_parity or state_parity" > gpurun_out/pytest_iter.log 2>&1
tail -2 gpurun_out/pytest_iter.log
python bench.py --config 4 --steps 10 --warmup 3 --no-cpu --no-srab > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err
python bench.py --config 5 --steps 5 --warmup 3 --no-cpu --no-srab > gpurun_out/bench_c5.json 2>gpurun_out/bench_c5.err
tail -2 gpurun_out/bench_c5.err
