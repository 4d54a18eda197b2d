cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_t55.log 2>&1; echo rc=$? >> gpurun_out/r2_t55.log
timeout 900 python bench.py --config c2 --math ffma --no-cpu --no-parametric --no-scaling --steps 5 > gpurun_out/r2_b55_c2f.json 2> gpurun_out/r2_b55_c2f.err
timeout 1200 python bench.py --config c3 --math ffma --no-cpu --no-parametric --no-scaling --steps 3 > gpurun_out/r2_b55_c3f.json 2> gpurun_out/r2_b55_c3f.err
