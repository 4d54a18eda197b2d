cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ffma_chain.py -q -p no:cacheprovider > gpurun_out/r2_t51.log 2>&1; echo rc=$? >> gpurun_out/r2_t51.log
timeout 300 python tools/single_chain.py 8 5 c4 ffma > gpurun_out/r2_sc51.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_train_ffma -s 2 -c 1 -o gpurun_out/r2_51_ffma -f python tools/single_chain.py 8 2 c4 ffma > gpurun_out/r2_51_ncu.log 2>&1
