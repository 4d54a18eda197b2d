cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
ECCO_WIDE_ST_ASYNC=1 timeout 1500 $CS --tool racecheck --print-limit 30 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_learned.py -k "wide_chain_within" > gpurun_out/r2_s88_race.log 2>&1
ECCO_WIDE_ST_ASYNC=1 timeout 1200 $CS --tool memcheck --print-limit 30 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_learned.py -k "wide_chain_within" > gpurun_out/r2_s88_mem.log 2>&1
ECCO_WIDE_ST_ASYNC=1 timeout 600 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_learned.py -k "wide_chain" > gpurun_out/r2_s88_plain.log 2>&1
