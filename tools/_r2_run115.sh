cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_ffma_chain.py tests/test_gpu_learned.py tests/test_gpu_decisions.py tests/test_gpu_multirank.py > gpurun_out/r2_t115.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r2_t115.txt 2>&1
timeout 1500 python bench.py --math ffma --no-parametric --no-cpu --no-e2e --no-probes --no-scaling --steps 3 > gpurun_out/r2_b115_c4f.json 2> gpurun_out/r2_b115_c4f.err
timeout 900 python bench.py --config c3 --math ffma --no-parametric --no-scaling --no-cpu --no-probes > gpurun_out/r2_b115_c3f.json 2> gpurun_out/r2_b115_c3f.err
timeout 600 python bench.py --no-parametric --no-cpu --no-probes --no-scaling --no-parity > gpurun_out/r2_b115_c4.json 2> gpurun_out/r2_b115_c4.err
SANITIZE_ONLY=learned bash tools/sanitize.sh gpurun_out/sanitize115
