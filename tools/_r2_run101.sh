cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_ffma_chain.py -k eval_matrix > gpurun_out/r2_t101.txt 2>&1
for u in 2 8 16; do
ECCO_FE_UNROLL=$u timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_ffma_chain.py -k "eval_matrix and 1-1-1" >> gpurun_out/r2_t101.txt 2>&1
ECCO_FE_UNROLL=$u timeout 1500 python bench.py --math ffma --no-parametric --no-cpu --no-e2e --no-probes --no-scaling --steps 3 > gpurun_out/r2_b101_c4f_$u.json 2> gpurun_out/r2_b101_c4f_$u.err
done
