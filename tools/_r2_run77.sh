cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ffma_chain.py tests/test_gpu_multirank.py -q -p no:cacheprovider -k "hidden_tiles or exact" > gpurun_out/r2_t77.log 2>&1; echo rc=$? >> gpurun_out/r2_t77.log
timeout 900 python bench.py --config c3 --math ffma --no-cpu --no-parametric --no-scaling --no-e2e --no-probes --steps 3 > gpurun_out/r2_b77_c3f.json 2> gpurun_out/r2_b77_c3f.err
timeout 2400 python bench.py --math ffma --no-parametric --no-cpu --no-e2e --no-probes --steps 3 > gpurun_out/r2_b77_c4f.json 2> gpurun_out/r2_b77_c4f.err
