cd $GRAFT_REPO_ROOT
./oracle/_ref/dropin_learned_test 1 6 > gpurun_out/r2_t5_dropin.log 2>&1; echo rc=$? >> gpurun_out/r2_t5_dropin.log
./oracle/_ref/dropin_learned_test 2 6 >> gpurun_out/r2_t5_dropin.log 2>&1; echo rc=$? >> gpurun_out/r2_t5_dropin.log
timeout 600 python -m pytest tests/test_gpu_parametric.py tests/test_gpu_sim.py -q -p no:cacheprovider > gpurun_out/r2_t5_param.log 2>&1; echo rc=$? >> gpurun_out/r2_t5_param.log
bash tools/sanitize.sh gpurun_out/r2_sanitize > gpurun_out/r2_sanitize.out 2>&1
