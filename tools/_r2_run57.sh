cd $GRAFT_REPO_ROOT
timeout 1800 python bench.py > gpurun_out/r2_b57_c4.json 2> gpurun_out/r2_b57_c4.err
timeout 1200 python bench.py --config c5 --no-parametric --no-scaling --steps 3 > gpurun_out/r2_b57_c5.json 2> gpurun_out/r2_b57_c5.err
timeout 900 python bench.py --config c2 --no-cpu --no-parametric --no-scaling > gpurun_out/r2_b57_c2.json 2> gpurun_out/r2_b57_c2.err
timeout 900 python bench.py --config c3 --no-cpu --no-parametric --no-scaling > gpurun_out/r2_b57_c3.json 2> gpurun_out/r2_b57_c3.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_b57_ref.json 2> gpurun_out/r2_b57_ref.err
