cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_learned.py tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/r2_t40.log 2>&1; echo rc=$? >> gpurun_out/r2_t40.log
timeout 300 python tools/single_chain.py 8 3 c5 >> gpurun_out/r2_t40.log 2>&1
timeout 1500 python bench.py --config c5 --no-parametric --no-scaling --no-cpu --steps 3 > gpurun_out/r2_b40_c5.json 2> gpurun_out/r2_b40_c5.err; echo rc=$? >> gpurun_out/r2_b40_c5.err
