#!/bin/bash
# Round-2 evidence (B200_PROFILING.md recipe), run on the GPU box:
#   launch lists (gpu__time_duration + DRAM bytes per launch) of C2, C3, C4, C5
#   and ncu --set full captures of the BetaE (C3), fusion (C4) and sharded (C5)
#   kernels. Usage: bash tools/profile_r02.sh [tag]
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras --profile-steps 1"
for CFG in c2 c3 c4 c5; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -s 400 -c 200 --csv --log-file $OUT/${CFG}_launches.csv \
      $B --config $CFG > /dev/null 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:"beta_prep|beta_entity_adam|stream_kernel|tc_gemm_tma" -s 60 -c 8 \
    -o $OUT/c3_full $B --config c3 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:"fuse|tc_gemm_tma" -s 60 -c 8 -o $OUT/c4_full $B --config c4 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:"shard_score|entity_adam|shard_anchor_pack|shard_grad_pack" -s 20 -c 6 \
    -o $OUT/c5_full $B --config c5 > /dev/null 2>&1
ls -la $OUT
