cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_t116.log 2>&1; echo rc=$? >> gpurun_out/r2_t116.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> gpurun_out/r2_t116.log 2>&1
timeout 1800 python bench.py > gpurun_out/r2_b116_c4.json 2> gpurun_out/r2_b116_c4.err; echo rc=$? >> gpurun_out/r2_b116_c4.err
