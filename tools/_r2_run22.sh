cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_learned.py -q -p no:cacheprovider -x > gpurun_out/r2_t22.log 2>&1; echo rc=$? >> gpurun_out/r2_t22.log
timeout 1800 python bench.py --config c5 --no-parametric --no-scaling --no-cpu --steps 3 > gpurun_out/r2_b22_c5.json 2> gpurun_out/r2_b22_c5.err
