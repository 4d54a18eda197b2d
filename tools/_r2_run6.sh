cd $GRAFT_REPO_ROOT
ECCO_DROPIN_VERBOSE=1 ./oracle/_ref/dropin_learned_test 1 2 0 > gpurun_out/r2_t6_dropin.log 2>&1
