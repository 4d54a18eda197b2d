cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_ffma_chain.py tests/test_gpu_multirank.py > gpurun_out/r2_t104.txt 2>&1
for v in 0 1; do
ECCO_FE_PERSIST=$v timeout 1500 python bench.py --math ffma --no-parametric --no-cpu --no-e2e --no-probes --no-scaling --steps 3 > gpurun_out/r2_b104_c4f_$v.json 2> gpurun_out/r2_b104_c4f_$v.err
done
timeout 2400 python bench.py --math ffma --no-parametric --no-cpu --no-e2e --no-probes --steps 3 > gpurun_out/r2_b104_c4f_scaling.json 2> gpurun_out/r2_b104_c4f_scaling.err
