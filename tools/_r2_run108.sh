cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_ffma_chain.py > gpurun_out/r2_t108.txt 2>&1
timeout 300 python tools/single_chain.py 8 5 c4 ffma > gpurun_out/r2_s108.txt 2>&1
timeout 900 python bench.py --config c2 --math ffma --no-parametric --no-scaling --no-cpu --no-probes > gpurun_out/r2_b108_c2f.json 2> gpurun_out/r2_b108_c2f.err
