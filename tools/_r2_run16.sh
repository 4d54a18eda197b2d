cd $GRAFT_REPO_ROOT
for cfg in "8 2" "12 4" "16 6"; do
  set -- $cfg
  ECCO_RESERVE_SMS=$1 ECCO_FETCH_CTAS=$2 timeout 900 python bench.py --no-parametric --no-scaling --no-cpu --no-probes --no-parity --steps 5 > gpurun_out/r2_b16_$1_$2.json 2> gpurun_out/r2_b16_$1_$2.err
done
ECCO_E2E_TRACE=1 timeout 900 python bench.py --no-parametric --no-scaling --no-cpu --no-probes --no-parity --steps 5 --e2e-full-rings > gpurun_out/r2_b16_full.json 2> gpurun_out/r2_b16_full.err
