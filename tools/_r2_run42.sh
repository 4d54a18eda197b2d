cd $GRAFT_REPO_ROOT
for r in 6 8 12 16; do
  ECCO_RESERVE_SMS=$r timeout 900 python bench.py --no-parametric --no-scaling --no-cpu --no-probes --no-parity --no-e2e --steps 6 > gpurun_out/r2_b42_$r.json 2> gpurun_out/r2_b42_$r.err
done
