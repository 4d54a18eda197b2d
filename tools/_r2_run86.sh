cd $GRAFT_REPO_ROOT
bash tools/sanitize.sh gpurun_out/r2_s86 > /dev/null 2>&1
