cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/r2_b41_c5.err
timeout 1500 python bench.py --config c5 --no-parametric --no-scaling --no-cpu --steps 3 > gpurun_out/r2_b41_c5.json 2>> gpurun_out/r2_b41_c5.err; echo rc=$? >> gpurun_out/r2_b41_c5.err
