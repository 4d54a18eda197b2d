cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ffma_chain.py tests/test_gpu_learned.py -q -p no:cacheprovider > gpurun_out/r2_t78.log 2>&1; echo rc=$? >> gpurun_out/r2_t78.log
timeout 900 python bench.py --config c3 --math ffma --no-cpu --no-parametric --no-scaling --no-e2e --no-probes --steps 3 > gpurun_out/r2_b78_c3f.json 2> gpurun_out/r2_b78_c3f.err
