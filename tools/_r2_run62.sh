cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ffma_chain.py tests/test_gpu_wide_eval.py -q -p no:cacheprovider > gpurun_out/r2_t62.log 2>&1; echo rc=$? >> gpurun_out/r2_t62.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool racecheck --print-limit 20 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_ffma_chain.py -k "unequal" > gpurun_out/r2_s62_ffma_race.log 2>&1
timeout 900 $CS --tool racecheck --print-limit 20 python -m pytest -q -p no:cacheprovider -m gpu -x tests/test_gpu_wide_eval.py -k "logits and odd or pairs_equal or regime and 2" > gpurun_out/r2_s62_wide_race.log 2>&1
