cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_learned.py -q -p no:cacheprovider -x > gpurun_out/r2_t21.log 2>&1; echo rc=$? >> gpurun_out/r2_t21.log
timeout 900 python bench.py --no-parametric --no-scaling --no-cpu --no-parity --steps 10 > gpurun_out/r2_b21.json 2> gpurun_out/r2_b21.err
