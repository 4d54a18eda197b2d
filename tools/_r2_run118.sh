cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --impl reference > gpurun_out/r2_b118_c4_ref.json 2> gpurun_out/r2_b118_c4_ref.err; echo rc=$? >> gpurun_out/r2_b118_c4_ref.err
timeout 1200 bash tools/profile.sh r2j k_eval_pair > gpurun_out/r2j_prof.out 2>&1; echo rc=$? >> gpurun_out/r2j_prof.out
