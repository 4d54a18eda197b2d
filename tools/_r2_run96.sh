cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_ffma_chain.py tests/test_gpu_learned.py > gpurun_out/r2_t96.txt 2>&1
for t in 64 32 128 100000; do
ECCO_PAIR_TILE=$t timeout 1500 python bench.py --math ffma --no-parametric --no-cpu --no-e2e --no-probes --no-scaling --steps 3 > gpurun_out/r2_b96_c4f_$t.json 2> gpurun_out/r2_b96_c4f_$t.err
done
ECCO_PAIR_TILE=64 timeout 900 python bench.py --config c3 --math ffma --no-parametric --no-scaling --no-cpu --no-probes > gpurun_out/r2_b96_c3f.json 2> gpurun_out/r2_b96_c3f.err
