cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_learned.py -q -p no:cacheprovider -k "wide" > gpurun_out/r2_t37.log 2>&1; echo rc=$? >> gpurun_out/r2_t37.log
OUT=gpurun_out/sanitize_wide; mkdir -p $OUT; : > $OUT/summary.txt
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  ECCO_WIDE_ST_ASYNC=1 timeout 1200 $CS --tool $tool --target-processes all --print-limit 50 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_learned.py -k "wide_chain_is_one or (wide_chain_within and 1024)" > $OUT/${tool}_st_async.log 2>&1
  echo "$tool st_async rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $OUT/${tool}_st_async.log | tr '\n' ';') $(grep -h 'passed\|failed' $OUT/${tool}_st_async.log | tail -1)" >> $OUT/summary.txt
done
for tool in synccheck racecheck; do
  timeout 1200 $CS --tool $tool --target-processes all --print-limit 50 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_learned.py -k "wide_chain_is_one or (wide_chain_within and 1024)" > $OUT/${tool}_bulk.log 2>&1
  echo "$tool bulk rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $OUT/${tool}_bulk.log | tr '\n' ';') $(grep -h 'passed\|failed' $OUT/${tool}_bulk.log | tail -1)" >> $OUT/summary.txt
done
