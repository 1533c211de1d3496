#!/bin/bash
# Profiling recipe (B200_PROFILING.md): launch list + full captures of the top kernels.
# Usage (on the GPU box): bash tools/profile_run.sh <tag>
set -x
TAG=${1:-r01}
CFG=${2:-c2}
mkdir -p gpurun_out
python bench.py --config $CFG --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 130 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --config $CFG --steps 3 --warmup 3 \
    --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"tc_gemm_kernel|entity_adam|loss_fwd" \
    -s 12 -c 6 -o gpurun_out/${TAG}_full python bench.py --config $CFG --steps 3 --warmup 3 \
    --no-cpu-baseline --profile-steps 1 > /dev/null 2>&1
ls -la gpurun_out
