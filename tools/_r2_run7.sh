cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_t7_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2_t7_gpu.log
python tools/param_probe.py all 5 > gpurun_out/r2_param_probe.json 2>&1
for k in k1:k_p_eval_matrix k2:k_p_trajectories k3:k_p_profile; do
  a=${k%%:*}; n=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$n -s 1 -c 1 -o gpurun_out/r2_$a -f python tools/param_probe.py $a 1 > gpurun_out/r2_ncu_$a.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-parametric --no-scaling --no-parity > gpurun_out/r2_launches_c4.log 2>&1
