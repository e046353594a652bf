export CUDA_LAUNCH_BLOCKING=1
for mesh in 1 0; do MESH=$mesh REPS=2 timeout 120 python scripts/one_rhs_launch.py > gpurun_out/one_$mesh.log 2>&1; echo "mesh $mesh rc=$?"; tail -1 gpurun_out/one_$mesh.log; done
