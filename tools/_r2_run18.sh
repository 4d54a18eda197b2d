cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_train_chain -s 3 -c 1 -o gpurun_out/r2_chain1 -f python tools/single_chain.py 2 2 > gpurun_out/r2_ncu_chain1.log 2>&1
