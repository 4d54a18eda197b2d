cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_ffma_chain.py tests/test_gpu_learned.py tests/test_gpu_decisions.py > gpurun_out/r2_t93.txt 2>&1
for v in 0 1; do
ECCO_FFMA_FUSED_EVAL=$v timeout 900 python bench.py --config c3 --math ffma --no-parametric --no-scaling --no-cpu --no-probes > gpurun_out/r2_b93_c3f_$v.json 2> gpurun_out/r2_b93_c3f_$v.err
ECCO_FFMA_FUSED_EVAL=$v timeout 1500 python bench.py --math ffma --no-parametric --no-cpu --no-e2e --no-probes --no-scaling --steps 3 > gpurun_out/r2_b93_c4f_$v.json 2> gpurun_out/r2_b93_c4f_$v.err
done
