cd $GRAFT_REPO_ROOT
for n in 4 8 12; do
  ECCO_FETCH_CTAS=$n timeout 900 python bench.py --no-cpu --no-parametric --no-scaling --no-probes --no-parity --steps 4 > gpurun_out/r2_b82_f$n.json 2> gpurun_out/r2_b82_f$n.err
done
