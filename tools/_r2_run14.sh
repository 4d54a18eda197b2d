cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_abi.py -q -p no:cacheprovider -x > gpurun_out/r2_t14.log 2>&1; echo rc=$? >> gpurun_out/r2_t14.log
timeout 1200 python bench.py --no-parametric --no-scaling --no-cpu > gpurun_out/r2_b14_c4.json 2> gpurun_out/r2_b14_c4.err
echo rc=$? >> gpurun_out/r2_b14_c4.err
