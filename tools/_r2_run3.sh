cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-parametric --no-scaling > gpurun_out/r2_b3_c3.json 2> gpurun_out/r2_b3_c3.err
echo rc=$? >> gpurun_out/r2_b3_c3.err
timeout 1200 python bench.py > gpurun_out/r2_b3_c4.json 2> gpurun_out/r2_b3_c4.err
echo rc=$? >> gpurun_out/r2_b3_c4.err
