cd $GRAFT_REPO_ROOT
ECCO_WIDE_TRACE=1 timeout 300 python tools/single_chain.py 2 1 c5 > gpurun_out/r2_t28.log 2>&1; echo rc=$? >> gpurun_out/r2_t28.log
timeout 300 python tools/single_chain.py 8 3 c5 >> gpurun_out/r2_t28.log 2>&1; echo rc=$? >> gpurun_out/r2_t28.log
timeout 600 python -m pytest tests/test_gpu_learned.py -q -p no:cacheprovider -k "wide or detection" >> gpurun_out/r2_t28.log 2>&1; echo rc=$? >> gpurun_out/r2_t28.log
