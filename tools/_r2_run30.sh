cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_learned.py -q -p no:cacheprovider -k "wide or detection" > gpurun_out/r2_t30.log 2>&1; echo rc=$? >> gpurun_out/r2_t30.log
timeout 1500 python bench.py --config c5 --no-parametric --no-scaling --no-cpu --steps 3 > gpurun_out/r2_b30_c5.json 2> gpurun_out/r2_b30_c5.err; echo rc=$? >> gpurun_out/r2_b30_c5.err
