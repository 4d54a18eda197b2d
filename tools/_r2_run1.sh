cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_t1_smi.txt 2>&1
lscpu > gpurun_out/r2_lscpu.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_fused_eval.py tests/test_gpu_decisions.py tests/test_gpu_learned.py -k "multi_tile or bench_shape or decisions" -q -s -p no:cacheprovider > gpurun_out/r2_t1.log 2>&1
echo rc=$? >> gpurun_out/r2_t1.log
