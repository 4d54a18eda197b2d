cd $GRAFT_REPO_ROOT
bash tools/ab.sh python tools/single_chain.py 8 5 c4 ffma > gpurun_out/r2_ab109_chain.txt 2>&1
bash tools/ab.sh bash -c "python bench.py --config c2 --math ffma --no-parametric --no-scaling --no-cpu --no-probes --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d[\"ms_per_step\"])'" > gpurun_out/r2_ab109_c2.txt 2>&1
