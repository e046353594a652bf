timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rhs_parity or state_parity" > gpurun_out/pytest_iter.log 2>&1
tail -1 gpurun_out/pytest_iter.log
MRAB_OVERLAP=1 python bench.py --steps 100 --warmup 5 --no-cpu --no-srab > gpurun_out/bench_ov.json 2>/dev/null
python bench.py --steps 100 --warmup 5 --no-cpu --no-srab > gpurun_out/bench_noov.json 2>/dev/null
MRAB_OVERLAP=1 MRAB_TMA=1 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-srab > gpurun_out/bench_ov_tma.json 2>/dev/null
MRAB_TMA=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "rhs_parity or state_parity or full3" > gpurun_out/pytest_tma.log 2>&1
tail -1 gpurun_out/pytest_tma.log
