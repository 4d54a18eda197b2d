cd $GRAFT_REPO_ROOT
python tools/single_chain.py 8 5 > gpurun_out/r2_single_chain.txt 2>&1
python tools/single_chain.py 1 20 >> gpurun_out/r2_single_chain.txt 2>&1
ECCO_LIB_PATH=$GRAFT_REPO_ROOT/paper_2512_11727_b200/libecco_b200_trace.so ECCO_CHAIN_TRACE=1 python tools/single_chain.py 2 1 > gpurun_out/r2_single_chain_trace.txt 2>&1
