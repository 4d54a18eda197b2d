cd $GRAFT_REPO_ROOT
timeout 600 python tools/param_window_probe.py c3 4 > gpurun_out/r2_pw70_c3.json 2> gpurun_out/r2_pw70_c3.err
