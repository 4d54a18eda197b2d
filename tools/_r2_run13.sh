cd $GRAFT_REPO_ROOT
ECCO_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c3 --steps 3 --warmup 3 > gpurun_out/r2_b13_c3_w2.json 2> gpurun_out/r2_b13_c3_w2.err
echo rc=$? >> gpurun_out/r2_b13_c3_w2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 --ref-budget 4 > gpurun_out/r2_b13_ref.json 2> gpurun_out/r2_b13_ref.err
