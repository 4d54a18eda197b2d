cd $GRAFT_REPO_ROOT
timeout 1200 python tools/decisions_probe.py c3 3 > gpurun_out/r2_decisions_c3.json 2> gpurun_out/r2_decisions_c3.err
timeout 900 python bench.py --config c2 --math ffma --no-parametric --no-scaling > gpurun_out/r2_b9_c2_ffma.json 2> gpurun_out/r2_b9_c2_ffma.err
timeout 900 python bench.py --config c3 --math ffma --no-parametric --no-scaling > gpurun_out/r2_b9_c3_ffma.json 2> gpurun_out/r2_b9_c3_ffma.err
timeout 900 python bench.py --config c3 --no-parametric --no-scaling > gpurun_out/r2_b9_c3.json 2> gpurun_out/r2_b9_c3.err
timeout 900 python bench.py --config c2 --no-parametric --no-scaling > gpurun_out/r2_b9_c2.json 2> gpurun_out/r2_b9_c2.err
timeout 1500 python bench.py --config c5 --no-parametric --no-scaling --steps 3 > gpurun_out/r2_b9_c5.json 2> gpurun_out/r2_b9_c5.err
