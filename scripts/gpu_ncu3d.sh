# ncu --set full capture of the two passes of the 3-D RHS on one mesh (after a plain run)
export CFG=${CFG:-4} MESH=${MESH:-1} KERNEL=0 REPS=1
python scripts/one_rhs_launch.py > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_flux3|k_rhs3d|k_div3' -c 2 -f -o gpurun_out/${OUT:-prof3d} python scripts/one_rhs_launch.py > gpurun_out/ncu_run.log 2>&1
echo "ncu rc $?"; tail -3 gpurun_out/ncu_run.log
