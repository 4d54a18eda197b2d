cd $GRAFT_REPO_ROOT
timeout 300 python tools/wide_err.py 1024 > gpurun_out/r2_t29.log 2>&1; echo rc=$? >> gpurun_out/r2_t29.log
timeout 300 python tools/wide_err.py 512 >> gpurun_out/r2_t29.log 2>&1; echo rc=$? >> gpurun_out/r2_t29.log
