cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_learned.py -q -p no:cacheprovider -x -k "sampled or fetch" > gpurun_out/r2_t17.log 2>&1; echo rc=$? >> gpurun_out/r2_t17.log
timeout 900 python bench.py --no-parametric --no-scaling --no-cpu --no-probes --no-parity --steps 5 > gpurun_out/r2_b17.json 2> gpurun_out/r2_b17.err
