cd $GRAFT_REPO_ROOT
for r in 12 20 28 40; do
  ECCO_RESERVE_SMS=$r timeout 900 python bench.py --no-parametric --no-scaling --no-cpu --no-probes --no-parity --steps 6 > gpurun_out/r2_b20_$r.json 2> gpurun_out/r2_b20_$r.err
done
