cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ffma_chain.py tests/test_gpu_learned.py -q -p no:cacheprovider > gpurun_out/r2_t91.log 2>&1; echo rc=$? >> gpurun_out/r2_t91.log
timeout 900 python bench.py --config c3 --math ffma --no-cpu --no-parametric --no-scaling --no-e2e --no-probes --no-parity --steps 3 > gpurun_out/r2_b91.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/r2_b91.json').read().strip().splitlines()[-1])
print(round(d['ms_per_step'],2), d['kernels']['EVAL_MATRIX'], d['kernels']['EVAL_PAIRS'])" >> gpurun_out/r2_t91.log
