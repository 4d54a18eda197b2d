cd $GRAFT_REPO_ROOT
timeout 1800 python bench.py --no-parametric --no-cpu > gpurun_out/r2_b39_c4.json 2> gpurun_out/r2_b39_c4.err; echo rc=$? >> gpurun_out/r2_b39_c4.err
