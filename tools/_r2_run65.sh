cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --config c5 --no-cpu --no-parametric --no-scaling --no-probes --no-parity --no-regroup --steps 3 > gpurun_out/r2_b65_c5.json 2> gpurun_out/r2_b65_c5.err
