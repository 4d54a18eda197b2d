cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_t79.log 2>&1; echo rc=$? >> gpurun_out/r2_t79.log
