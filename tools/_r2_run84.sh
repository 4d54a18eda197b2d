cd $GRAFT_REPO_ROOT
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:k_fetch_rows -c 6 --log-file gpurun_out/r2_84_fetch.csv python bench.py --no-cpu --no-parametric --no-scaling --no-probes --no-parity --steps 1 --warmup 3 > gpurun_out/r2_84.log 2>&1
