cd $GRAFT_REPO_ROOT
SANITIZE_ONLY=ffma_chain bash tools/sanitize.sh gpurun_out/r2_s61 > /dev/null 2>&1
SANITIZE_ONLY=wide_eval bash tools/sanitize.sh gpurun_out/r2_s61w > /dev/null 2>&1
ECCO_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-parametric > gpurun_out/r2_b61_gloo2.json 2> gpurun_out/r2_b61_gloo2.err; echo rc=$? >> gpurun_out/r2_b61_gloo2.err
