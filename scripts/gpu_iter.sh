# one build -> measure iteration on the GPU box (parity subset, bench, ncu of the 2-D RHS)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rhs_parity or state_parity" > gpurun_out/pytest_iter.log 2>&1
python bench.py --steps 100 --warmup 5 --config ${CFG:-3} --no-cpu > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err
if [ -n "$NCU" ]; then
python bench.py --steps 3 --warmup 3 --no-srab --no-cpu > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:${NCU} -s ${NCU_SKIP:-12} -c 2 -o gpurun_out/prof_iter python bench.py --steps 3 --warmup 3 --no-srab --no-cpu > gpurun_out/ncu_full.log 2>&1
fi
tail -2 gpurun_out/pytest_iter.log
