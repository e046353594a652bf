timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "not config4 and not config5" > gpurun_out/pytest_iter.log 2>&1
tail -1 gpurun_out/pytest_iter.log
rm -f gpurun_out/sweep.txt; VARIANTS=0 bash scripts/k2d_sweep.sh > /dev/null 2>&1; cat gpurun_out/sweep.txt
MRAB_STREAM=0 python bench.py --steps 100 --warmup 5 --no-cpu --no-srab > gpurun_out/bench_nostream.json 2> /dev/null
python bench.py --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err
