timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_iter.log 2>&1
tail -2 gpurun_out/pytest_iter.log
python bench.py --steps 100 --warmup 5 --config 3 --no-cpu > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err
MRAB_OVERLAP=0 python bench.py --steps 100 --warmup 5 --config 3 --no-cpu --no-srab > gpurun_out/bench_noov.json 2> gpurun_out/bench_noov.err
python bench.py --steps 100 --warmup 5 --config 2 --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -3 gpurun_out/bench_iter.err
