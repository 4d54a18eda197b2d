cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_ffma_chain.py -q -p no:cacheprovider > gpurun_out/r2_t75.log 2>&1; echo rc=$? >> gpurun_out/r2_t74.log
timeout 2400 python bench.py --math ffma --no-parametric --no-cpu --no-e2e --no-probes --steps 3 > gpurun_out/r2_b75_c4f.json 2> gpurun_out/r2_b75_c4f.err
