cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ffma_chain.py -q -p no:cacheprovider -k hidden_tiles > gpurun_out/r2_t69.log 2>&1; echo rc=$? >> gpurun_out/r2_t69.log
timeout 900 python bench.py --config c3 --math ffma --no-cpu --no-parametric --no-scaling --no-e2e --no-probes --steps 3 > gpurun_out/r2_b69_c3f.json 2> gpurun_out/r2_b69_c3f.err
