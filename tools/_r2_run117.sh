cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_t117.log 2>&1; echo rc=$? >> gpurun_out/r2_t117.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> gpurun_out/r2_t117.log 2>&1
timeout 1800 python bench.py > gpurun_out/r2_b117_c4.json 2> gpurun_out/r2_b117_c4.err; echo rc=$? >> gpurun_out/r2_b117_c4.err
for r in 10 14; do ECCO_RESERVE_SMS=$r timeout 900 python bench.py > gpurun_out/r2_b117_c4_res$r.json 2> gpurun_out/r2_b117_c4_res$r.err; done
