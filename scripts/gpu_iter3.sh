# 3-D iteration: parity + overlap tests, then config 4/5 bench lines with the overlapped and the serial schedule
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "${PT_K:-overlapped or state or rhs}" > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_iter.log
tail -8 gpurun_out/pytest_iter.log
for c in ${BENCH_CFGS:-4 5}; do
  for ov in 1 0; do
    MRAB_OVERLAP3D=$ov timeout 600 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu --no-srab --no-secondary > gpurun_out/bench_c${c}_ov$ov.json 2> gpurun_out/bench_c${c}_ov$ov.err
    echo "config $c overlap $ov"; python scripts/show_bench.py gpurun_out/bench_c${c}_ov$ov.json 2>/dev/null || tail -5 gpurun_out/bench_c${c}_ov$ov.err
  done
done
CFG=4 timeout 300 python scripts/trace_step3d.py > gpurun_out/trace3d_c4.txt 2>&1; tail -30 gpurun_out/trace3d_c4.txt
CFG=5 timeout 300 python scripts/trace_step3d.py > gpurun_out/trace3d_c5.txt 2>&1; tail -70 gpurun_out/trace3d_c5.txt
