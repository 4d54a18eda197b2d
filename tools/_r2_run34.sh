cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_train_wide -s 4 -c 1 -o gpurun_out/r2_wide1 -f python tools/single_chain.py 8 1 c5 > gpurun_out/r2_wide1.log 2>&1
echo rc=$? >> gpurun_out/r2_wide1.log
