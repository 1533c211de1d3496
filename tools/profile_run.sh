#!/bin/bash
# Profiling recipe (B200_PROFILING.md): launch list of one step + full captures
# of the top kernels. Usage (on the GPU box): bash tools/profile_run.sh <tag> [config] [kernel regex]
TAG=${1:-r01}
CFG=${2:-c2}
KRE=${3:-"tc_gemm_kernel|entity_adam|stream_kernel"}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 160 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --config $CFG --steps 3 --warmup 3 \
    --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"$KRE" \
    -s 12 -c 8 -o gpurun_out/${TAG}_full python bench.py --config $CFG --steps 3 --warmup 3 \
    --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
ls -la gpurun_out
