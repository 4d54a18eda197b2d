cd $GRAFT_REPO_ROOT
bash tools/ab.sh timeout 300 python tools/single_chain.py 8 5 c5 > gpurun_out/r2_ab47.txt 2>&1
