cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ffma_chain.py tests/test_gpu_learned.py -q -p no:cacheprovider > gpurun_out/r2_t58.log 2>&1; echo rc=$? >> gpurun_out/r2_t58.log
ECCO_FFMA_TRACE=1 timeout 300 python tools/single_chain.py 2 1 c4 ffma > gpurun_out/r2_sc58_trace.txt 2>&1
timeout 300 python tools/single_chain.py 8 5 c4 ffma > gpurun_out/r2_sc58.txt 2>&1
timeout 900 python bench.py --config c3 --no-cpu --no-parametric --no-scaling > gpurun_out/r2_b58_c3.json 2> gpurun_out/r2_b58_c3.err; echo rc=$? >> gpurun_out/r2_b58_c3.err
timeout 900 python bench.py --config c3 --math ffma --no-cpu --no-parametric --no-scaling --steps 3 > gpurun_out/r2_b58_c3f.json 2> gpurun_out/r2_b58_c3f.err; echo rc=$? >> gpurun_out/r2_b58_c3f.err
