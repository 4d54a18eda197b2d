cd $GRAFT_REPO_ROOT
timeout 900 python tools/decisions_probe.py c3 5 > gpurun_out/r2_dec63_c3.json 2> gpurun_out/r2_dec63_c3.err
timeout 1800 python tools/decisions_probe.py c4 3 > gpurun_out/r2_dec63_c4.json 2> gpurun_out/r2_dec63_c4.err
