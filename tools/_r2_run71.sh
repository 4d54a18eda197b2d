cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parametric.py tests/test_gpu_sim.py tests/test_reference_suite.py tests/test_dropin.py -q -p no:cacheprovider > gpurun_out/r2_t71.log 2>&1; echo rc=$? >> gpurun_out/r2_t71.log
timeout 600 python tools/param_window_probe.py c3 4 > gpurun_out/r2_pw71_c3.json 2> gpurun_out/r2_pw71_c3.err
timeout 600 python tools/param_window_probe.py c4 2 > gpurun_out/r2_pw71_c4.json 2> gpurun_out/r2_pw71_c4.err
