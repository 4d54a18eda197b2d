cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_learned.py tests/test_gpu_multirank.py -q -p no:cacheprovider -x > gpurun_out/r2_t38.log 2>&1; echo rc=$? >> gpurun_out/r2_t38.log
timeout 300 python tools/single_chain.py 8 3 c4 >> gpurun_out/r2_t38.log 2>&1
ECCO_NO_SERIAL_CHAIN=1 timeout 300 python tools/single_chain.py 8 3 c4 >> gpurun_out/r2_t38.log 2>&1
timeout 300 python tools/single_chain.py 64 2 c4 >> gpurun_out/r2_t38.log 2>&1
