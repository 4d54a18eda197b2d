cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_ffma_chain.py tests/test_gpu_learned.py tests/test_gpu_decisions.py tests/test_gpu_multirank.py > gpurun_out/r2_t107.txt 2>&1
timeout 300 python tools/single_chain.py 8 5 c4 ffma > gpurun_out/r2_s107.txt 2>&1
timeout 900 python bench.py --config c2 --math ffma --no-parametric --no-scaling --no-cpu --no-probes > gpurun_out/r2_b107_c2f.json 2> gpurun_out/r2_b107_c2f.err
timeout 900 python bench.py --config c3 --math ffma --no-parametric --no-scaling --no-cpu --no-probes > gpurun_out/r2_b107_c3f.json 2> gpurun_out/r2_b107_c3f.err
timeout 1500 python bench.py --math ffma --no-parametric --no-cpu --no-e2e --no-probes --no-scaling --steps 3 > gpurun_out/r2_b107_c4f.json 2> gpurun_out/r2_b107_c4f.err
