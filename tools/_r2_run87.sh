cd $GRAFT_REPO_ROOT
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export ECCO_WIDE_DBG_SKIPX=1; else unset ECCO_WIDE_DBG_SKIPX; fi
  echo "skipx=$v $(timeout 300 python tools/single_chain.py 8 3 c5 2>&1 | tail -1)" >> gpurun_out/r2_87.txt
done
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck; do
  ECCO_WIDE_ST_ASYNC=1 timeout 1200 $CS --tool $tool --print-limit 20 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_learned.py -k "wide_chain_within" > gpurun_out/r2_s87_$tool.log 2>&1
done
