cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py --math ffma --no-parametric --no-scaling --no-cpu --steps 3 > gpurun_out/r2_b67_c4f.json 2> gpurun_out/r2_b67_c4f.err
timeout 900 python bench.py --config c2 --no-parametric --no-scaling > gpurun_out/r2_b67_c2.json 2> gpurun_out/r2_b67_c2.err
timeout 900 python bench.py --config c3 --no-parametric --no-scaling > gpurun_out/r2_b67_c3.json 2> gpurun_out/r2_b67_c3.err
