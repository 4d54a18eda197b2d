cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2_t15_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2_t15_gpu.log
timeout 300 python __graft_entry__.py >> gpurun_out/r2_t15_gpu.log 2>&1
timeout 1800 python bench.py > gpurun_out/r2_b15_c4.json 2> gpurun_out/r2_b15_c4.err
echo rc=$? >> gpurun_out/r2_b15_c4.err
