#!/bin/bash
# Round profiling recipe (B200_PROFILING.md), run on the GPU box through gpurun:
#   tools/profile.sh TAG [KERNEL_REGEX...]
# -> gpurun_out/TAG_launches.csv   launch list of one bench step (gpu__time_duration, no clock control)
#    gpurun_out/TAG_<k>.ncu-rep    one --set full capture per kernel regex (with source)
set -u
tag=${1:-prof}
shift || true
cfg=${ECCO_PROFILE_CONFIG:-c4}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu --no-e2e --no-parametric --no-scaling --no-regroup \
    > gpurun_out/${tag}_launches.log 2>&1
for k in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/${tag}_${k} -f \
      python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu --no-e2e --no-parametric --no-scaling --no-regroup \
      > gpurun_out/${tag}_${k}.log 2>&1
done
