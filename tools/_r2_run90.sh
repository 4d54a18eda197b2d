cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ffma_chain.py tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/r2_t90.log 2>&1; echo rc=$? >> gpurun_out/r2_t90.log
