cd $GRAFT_REPO_ROOT
timeout 600 python tools/window_phases.py c2 4 > gpurun_out/r2_wp81_c2.json 2> gpurun_out/r2_wp81_c2.err
timeout 600 python tools/window_phases.py c3 4 > gpurun_out/r2_wp81_c3.json 2> gpurun_out/r2_wp81_c3.err
