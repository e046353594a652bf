# ncu full capture of one march-kernel launch (bg mesh of config 3) + PD sweep timing
python scripts/one_rhs_launch.py > gpurun_out/one.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rhs2d_m -c 1 -o gpurun_out/march1 -f python scripts/one_rhs_launch.py > gpurun_out/ncu_march.log 2>&1
tail -3 gpurun_out/ncu_march.log
for pd in 0 2 4 8; do
  MRAB_MARCH_PD=$pd REPS=10 python scripts/one_rhs_launch.py 2>&1 | tail -1 | sed "s/^/pd=$pd /"
done
MRAB_MARCH_L=64 REPS=10 python scripts/one_rhs_launch.py 2>&1 | tail -1 | sed "s/^/L=64 /"
MRAB_MARCH_CTAS=1 REPS=10 python scripts/one_rhs_launch.py 2>&1 | tail -1 | sed "s/^/ctas1 /"
