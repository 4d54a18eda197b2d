cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_t111.log 2>&1; echo rc=$? >> gpurun_out/r2_t111.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> gpurun_out/r2_t111.log 2>&1
timeout 1800 python bench.py > gpurun_out/r2_b111_c4.json 2> gpurun_out/r2_b111_c4.err; echo rc=$? >> gpurun_out/r2_b111_c4.err
timeout 900 python bench.py --config c2 --math ffma --no-parametric --no-scaling > gpurun_out/r2_b111_c2f.json 2> gpurun_out/r2_b111_c2f.err
timeout 900 python bench.py --config c3 --math ffma --no-parametric --no-scaling > gpurun_out/r2_b111_c3f.json 2> gpurun_out/r2_b111_c3f.err
SANITIZE_ONLY=ffma_chain bash tools/sanitize.sh gpurun_out/sanitize111
