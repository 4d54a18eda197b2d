cd $GRAFT_REPO_ROOT
for v in 2 3; do
ECCO_FE_BLOCKS=$v timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_ffma_chain.py -k "eval_matrix" > gpurun_out/r2_t106_$v.txt 2>&1
ECCO_FE_BLOCKS=$v timeout 1500 python bench.py --math ffma --no-parametric --no-cpu --no-e2e --no-probes --no-scaling --steps 3 > gpurun_out/r2_b106_c4f_$v.json 2> gpurun_out/r2_b106_c4f_$v.err
done
