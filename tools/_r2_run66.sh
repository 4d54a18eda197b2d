cd $GRAFT_REPO_ROOT
timeout 1500 bash tools/profile.sh r2h_c4 k_eval_pair
