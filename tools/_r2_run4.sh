cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_dropin.py tests/test_gpu_multirank.py -q -s -p no:cacheprovider > gpurun_out/r2_t4.log 2>&1
echo rc=$? >> gpurun_out/r2_t4.log
timeout 1200 python bench.py --no-parametric > gpurun_out/r2_b4_c4.json 2> gpurun_out/r2_b4_c4.err
echo rc=$? >> gpurun_out/r2_b4_c4.err
