cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_learned.py tests/test_gpu_multirank.py tests/test_gpu_decisions.py -q -p no:cacheprovider -x > gpurun_out/r2_t12.log 2>&1; echo rc=$? >> gpurun_out/r2_t12.log
timeout 300 python __graft_entry__.py >> gpurun_out/r2_t12.log 2>&1
python tools/single_chain.py 8 5 > gpurun_out/r2_single_chain12.txt 2>&1
timeout 1200 python bench.py --no-parametric --no-scaling --no-cpu > gpurun_out/r2_b12_c4.json 2> gpurun_out/r2_b12_c4.err
