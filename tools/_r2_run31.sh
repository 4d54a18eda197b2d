cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_t31.log 2>&1; echo rc=$? >> gpurun_out/r2_t31.log
timeout 300 python tools/single_chain.py 8 3 c5 >> gpurun_out/r2_t31.log 2>&1
timeout 1500 python bench.py --config c5 --no-parametric --no-scaling --no-cpu --steps 3 > gpurun_out/r2_b31_c5.json 2> gpurun_out/r2_b31_c5.err; echo rc=$? >> gpurun_out/r2_b31_c5.err
