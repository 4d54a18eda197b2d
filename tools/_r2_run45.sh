cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_wide_eval.py -x -q -p no:cacheprovider > gpurun_out/r2_t45_wide.log 2>&1; echo rc=$? >> gpurun_out/r2_t45_wide.log
timeout 900 python -m pytest tests/test_gpu_learned.py tests/test_gpu_fused_eval.py -q -p no:cacheprovider >> gpurun_out/r2_t45_wide.log 2>&1; echo rc=$? >> gpurun_out/r2_t45_wide.log
