cd $GRAFT_REPO_ROOT
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_l_hidden_ffma8 -s 20 -c 1 -o gpurun_out/r2_68_h8 -f python bench.py --math ffma --config c3 --steps 1 --warmup 3 --no-cpu --no-e2e --no-parametric --no-scaling --no-probes --no-parity > gpurun_out/r2_68.log 2>&1
