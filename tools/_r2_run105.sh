cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_ffma_chain.py tests/test_gpu_multirank.py > gpurun_out/r2_t105.txt 2>&1
timeout 2400 python bench.py --math ffma --no-parametric --no-cpu --no-probes --steps 3 > gpurun_out/r2_b105_c4f_scaling.json 2> gpurun_out/r2_b105_c4f_scaling.err
