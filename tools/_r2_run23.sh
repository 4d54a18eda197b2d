cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_t23_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2_t23_gpu.log
timeout 300 python __graft_entry__.py >> gpurun_out/r2_t23_gpu.log 2>&1
/usr/bin/time -v timeout 1800 python bench.py > gpurun_out/r2_b23_c4.json 2> gpurun_out/r2_b23_c4.err
echo rc=$? >> gpurun_out/r2_b23_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2_launches_c4b.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-parametric --no-scaling --no-parity --no-probes > gpurun_out/r2_launches_c4b.log 2>&1
