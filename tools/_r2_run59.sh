cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_train_ffma -s 2 -c 1 -o gpurun_out/r2_59_ffma -f python tools/single_chain.py 8 2 c4 ffma > gpurun_out/r2_59_ncu.log 2>&1
