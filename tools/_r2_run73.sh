cd $GRAFT_REPO_ROOT
timeout 2400 python bench.py --math ffma --no-parametric --no-cpu --no-e2e --no-probes --steps 3 > gpurun_out/r2_b73_c4f.json 2> gpurun_out/r2_b73_c4f.err
