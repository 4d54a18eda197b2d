cd $GRAFT_REPO_ROOT
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_p100_launches.csv \
  timeout 900 python bench.py --math ffma --steps 1 --warmup 3 --no-cpu --no-e2e --no-parametric --no-scaling --no-regroup --no-probes > gpurun_out/r2_p100_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_l_eval_ffma_fused -s 1002 -c 1 -o gpurun_out/r2_p100_fused_big -f \
  python bench.py --math ffma --steps 1 --warmup 3 --no-cpu --no-e2e --no-parametric --no-scaling --no-regroup --no-probes > gpurun_out/r2_p100_fused_big.log 2>&1
