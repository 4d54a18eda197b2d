cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "stag or ingest or fetch or swap or frames" > gpurun_out/r2_t83.log 2>&1; echo rc=$? >> gpurun_out/r2_t83.log
timeout 900 python bench.py --no-cpu --no-parametric --no-scaling --no-probes --no-parity --steps 4 > gpurun_out/r2_b83.json 2> gpurun_out/r2_b83.err
timeout 900 python bench.py --no-cpu --no-parametric --no-scaling --no-probes --no-parity --steps 4 > gpurun_out/r2_b83b.json 2> gpurun_out/r2_b83b.err
