cd $GRAFT_REPO_ROOT
ECCO_DEBUG=1 timeout 300 python -m pytest tests/test_gpu_learned.py -q -p no:cacheprovider -x -k "wide_chain_is_one" > gpurun_out/r2_t26.log 2>&1; echo rc=$? >> gpurun_out/r2_t26.log
