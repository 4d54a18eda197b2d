cd $GRAFT_REPO_ROOT
for c in c2 c3; do
  timeout 900 python bench.py --config $c --no-parametric --no-scaling > gpurun_out/r2_b19_$c.json 2> gpurun_out/r2_b19_$c.err
  timeout 900 python bench.py --config $c --math ffma --no-parametric --no-scaling > gpurun_out/r2_b19_${c}_ffma.json 2> gpurun_out/r2_b19_${c}_ffma.err
done
timeout 1800 python bench.py --config c5 --no-parametric --no-scaling --steps 3 > gpurun_out/r2_b19_c5.json 2> gpurun_out/r2_b19_c5.err
