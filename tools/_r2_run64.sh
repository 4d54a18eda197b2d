cd $GRAFT_REPO_ROOT
for n in 4 16 32; do
  ECCO_FETCH_CTAS=$n timeout 900 python bench.py --config c5 --no-cpu --no-parametric --no-scaling --no-probes --no-parity --no-regroup --steps 3 > gpurun_out/r2_b64_c5_f$n.json 2> gpurun_out/r2_b64_c5_f$n.err
done
