cd $GRAFT_REPO_ROOT
for v in 0 1 2; do
  ECCO_EVAL_DBG_SKIP=$v timeout 600 python tools/wide_eval_bench.py 2000 64 3 > /dev/null 2>&1
  ECCO_EVAL_DBG_SKIP=$v timeout 900 python -c "
import sys, json, time; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2512_11727_b200 as ecco
N,G=4000,256
ctx=ecco.Context(backend=ecco.LEARNED, math=ecco.TC_BF16, max_cameras=N, max_jobs=G, max_depth=2, feat_dim=512, hidden_dim=256, num_classes=16, minibatch=128, ring_frames=64, eval_samples=64)
rng=np.random.default_rng(0); ctx.set_cameras(np.round(rng.random((N,2)),1), np.full(N,8.192e6)); ctx.generate_frames(1)
ids=list(range(G)); ctx.seed_models(ids)
out=torch.empty((N,G),dtype=torch.float64,device='cuda'); cams=np.arange(N,dtype=np.int32)
ctx.eval_matrix_dev(ids,out.data_ptr(),cams=cams); ctx.synchronize()
ctx.profile(True)
for _ in range(3): ctx.eval_matrix_dev(ids,out.data_ptr(),cams=cams)
ctx.synchronize(); n,ms,fl,by=ctx.kernel_stat(ecco.KSTAT_EVAL_MATRIX)
print('skip=$v', round(ms/n,3), 'ms', round(fl/ms/1e9,1), 'TF/s')
" >> gpurun_out/r2_85.txt 2>&1
done
