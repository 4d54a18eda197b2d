cd $GRAFT_REPO_ROOT
timeout 1700 python -m pytest tests -m gpu -q -s -p no:cacheprovider -x --durations=15 > gpurun_out/r2_t2.log 2>&1
echo rc=$? >> gpurun_out/r2_t2.log
