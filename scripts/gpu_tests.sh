# GPU box: selected test files (TESTS), log to gpurun_out/
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout ${PT_TIMEOUT:-1700} python -m pytest ${TESTS:-tests -m gpu} -x -q -rA --durations=15 ${PT_K:+-k "$PT_K"} > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_sel.log
tail -40 gpurun_out/pytest_sel.log
