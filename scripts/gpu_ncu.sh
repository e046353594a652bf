# one ncu --set full capture of a kernel launched by scripts/one_rhs_launch.py (after a plain run)
# env: CFG, MESH, KERNEL (mrab_time_kernel id), KREGEX, OUT
export CFG=${CFG:-4} MESH=${MESH:-1} KERNEL=${KERNEL:-0} REPS=1
python scripts/one_rhs_launch.py > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_rhs3z} -c 1 -f -o gpurun_out/${OUT:-prof} python scripts/one_rhs_launch.py > gpurun_out/ncu_run.log 2>&1
echo "ncu rc $?"; tail -3 gpurun_out/ncu_run.log
