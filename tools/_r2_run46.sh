cd $GRAFT_REPO_ROOT
timeout 300 python tools/wide_eval_bench.py 2000 64 3 > gpurun_out/r2_w46.json 2> gpurun_out/r2_w46.err
timeout 300 python tools/wide_eval_bench.py 10000 500 1 > gpurun_out/r2_w46_full.json 2>> gpurun_out/r2_w46.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_eval_wide -s 1 -c 1 -o gpurun_out/r2_w46_eval_wide -f python tools/wide_eval_bench.py 1024 32 1 > gpurun_out/r2_w46_ncu.log 2>&1
timeout 1200 python bench.py --config c5 --no-cpu --no-parametric --no-scaling --steps 3 > gpurun_out/r2_b46_c5.json 2> gpurun_out/r2_b46_c5.err
