cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_wide_eval.py tests/test_gpu_fused_eval.py tests/test_gpu_learned.py -q -p no:cacheprovider > gpurun_out/r2_t49.log 2>&1; echo rc=$? >> gpurun_out/r2_t49.log
SANITIZE_ONLY=wide_eval bash tools/sanitize.sh gpurun_out/r2_s49 > /dev/null 2>&1
timeout 1200 python bench.py --config c5 --no-parametric --no-scaling --steps 3 > gpurun_out/r2_b49_c5.json 2> gpurun_out/r2_b49_c5.err
ECCO_PROFILE_CONFIG=c5 timeout 1200 bash tools/profile.sh r2h_c5
