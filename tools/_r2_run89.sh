cd $GRAFT_REPO_ROOT
ECCO_FFMA_HIDDEN16=1 timeout 600 python -m pytest tests/test_gpu_ffma_chain.py -q -p no:cacheprovider -k "hidden_tiles" > gpurun_out/r2_t89.log 2>&1; echo rc=$? >> gpurun_out/r2_t89.log
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export ECCO_FFMA_HIDDEN16=1; else unset ECCO_FFMA_HIDDEN16; fi
  timeout 900 python bench.py --config c3 --math ffma --no-cpu --no-parametric --no-scaling --no-e2e --no-probes --no-parity --steps 3 > gpurun_out/r2_b89_$v.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/r2_b89_$v.json').read().strip().splitlines()[-1])
print('h16=$v', round(d['ms_per_step'],2), d['kernels']['EVAL_MATRIX'])" >> gpurun_out/r2_89.txt
done
unset ECCO_FFMA_HIDDEN16
