cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_ffma_chain.py -k eval_matrix > gpurun_out/r2_t98.txt 2>&1
timeout 1500 python bench.py --math ffma --no-parametric --no-cpu --no-e2e --no-probes --no-scaling --steps 3 > gpurun_out/r2_b98_c4f.json 2> gpurun_out/r2_b98_c4f.err
