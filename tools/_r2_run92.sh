cd $GRAFT_REPO_ROOT
timeout 2400 python bench.py --math ffma --no-parametric --no-cpu --no-e2e --no-probes --steps 3 > gpurun_out/r2_b92_c4f.json 2> gpurun_out/r2_b92_c4f.err
timeout 900 python bench.py --config c2 --math ffma --no-parametric --no-scaling > gpurun_out/r2_b92_c2f.json 2> gpurun_out/r2_b92_c2f.err
timeout 900 python bench.py --config c3 --math ffma --no-parametric --no-scaling > gpurun_out/r2_b92_c3f.json 2> gpurun_out/r2_b92_c3f.err
