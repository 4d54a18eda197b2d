cd $GRAFT_REPO_ROOT
SANITIZE_ONLY=wide_eval bash tools/sanitize.sh gpurun_out/r2_s48 > /dev/null 2>&1
timeout 1200 python bench.py --config c5 --no-parametric --no-scaling --steps 3 > gpurun_out/r2_b48_c5.json 2> gpurun_out/r2_b48_c5.err
ECCO_PROFILE_CONFIG=c5 timeout 1200 bash tools/profile.sh r2h_c5
