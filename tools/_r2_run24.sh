cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2_t24_gpu.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider >> gpurun_out/r2_t24_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2_t24_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> gpurun_out/r2_t24_gpu.log 2>&1
timeout 1800 python bench.py > gpurun_out/r2_b24_c4.json 2> gpurun_out/r2_b24_c4.err; echo rc=$? >> gpurun_out/r2_b24_c4.err
