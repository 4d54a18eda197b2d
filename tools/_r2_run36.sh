cd $GRAFT_REPO_ROOT
OUT=gpurun_out/sanitize_wide; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  timeout 1200 $CS --tool $tool --target-processes all --print-limit 50 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_learned.py -k "wide_chain_is_one or (wide_chain_within and 1024)" > $OUT/${tool}.log 2>&1
  echo "$tool rc=$? $(grep -h 'ERROR SUMMARY' $OUT/${tool}.log | tr '\n' ';')" >> $OUT/summary.txt
done
