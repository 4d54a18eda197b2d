cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2_t8_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2_t8_gpu.log
python tools/param_probe.py all 10 > gpurun_out/r2_param_probe.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_p_eval_matrix -s 1 -c 1 -o gpurun_out/r2_k1b -f python tools/param_probe.py k1 1 > gpurun_out/r2_ncu_k1b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_p_trajectories -s 1 -c 1 -o gpurun_out/r2_k2 -f python tools/param_probe.py k2 1 > gpurun_out/r2_ncu_k2.log 2>&1
timeout 1200 python bench.py --no-parametric --no-scaling > gpurun_out/r2_b8_c4.json 2> gpurun_out/r2_b8_c4.err
