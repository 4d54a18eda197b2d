cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ffma_chain.py -x -q -p no:cacheprovider > gpurun_out/r2_t50.log 2>&1; echo rc=$? >> gpurun_out/r2_t50.log
timeout 900 python -m pytest tests/test_gpu_learned.py tests/test_gpu_decisions.py tests/test_gpu_multirank.py -q -p no:cacheprovider >> gpurun_out/r2_t50.log 2>&1; echo rc=$? >> gpurun_out/r2_t50.log
timeout 900 python bench.py --config c2 --math ffma --no-cpu --no-parametric --no-scaling --steps 5 > gpurun_out/r2_b50_c2f.json 2> gpurun_out/r2_b50_c2f.err
