cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2_t10_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2_t10_gpu.log
timeout 1200 python bench.py --no-parametric --no-scaling > gpurun_out/r2_b10_c4.json 2> gpurun_out/r2_b10_c4.err
