cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py --config c5 --no-parametric --no-scaling --no-cpu --steps 3 > gpurun_out/r2_b35_c5.json 2> gpurun_out/r2_b35_c5.err; echo rc=$? >> gpurun_out/r2_b35_c5.err
