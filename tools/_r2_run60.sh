cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ffma_chain.py -q -p no:cacheprovider > gpurun_out/r2_t60.log 2>&1; echo rc=$? >> gpurun_out/r2_t60.log
timeout 300 python tools/single_chain.py 8 5 c4 ffma > gpurun_out/r2_sc60.txt 2>&1
