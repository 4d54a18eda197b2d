cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_learned.py -q -p no:cacheprovider -x -k "wide_chain_is_one" > gpurun_out/r2_t25.log 2>&1; echo rc=$? >> gpurun_out/r2_t25.log
timeout 600 python -m pytest tests/test_gpu_learned.py -q -p no:cacheprovider -k "wide or detection" >> gpurun_out/r2_t25.log 2>&1; echo rc=$? >> gpurun_out/r2_t25.log
timeout 300 python tools/single_chain.py 8 3 c5 >> gpurun_out/r2_t25.log 2>&1; echo rc=$? >> gpurun_out/r2_t25.log
timeout 300 python tools/single_chain.py 8 3 c4 >> gpurun_out/r2_t25.log 2>&1; echo rc=$? >> gpurun_out/r2_t25.log
