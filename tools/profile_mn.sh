#!/bin/bash
# Evidence for the MN-major GEMM operands (run on the GPU box): launch lists of
# C2-C5 (time + DRAM bytes per launch), an ncu --set full capture of the C2
# GEMM launches (the weight-gradient levels read MN-major operands), and the
# C5 bench line. Usage: bash tools/profile_mn.sh [tag]
TAG=${1:-r02n}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python bench.py --config c5 --steps 100 --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras --profile-steps 1"
for CFG in c2 c3 c4 c5; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -s 400 -c 200 --csv --log-file $OUT/${CFG}_launches.csv \
      $B --config $CFG > /dev/null 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:"tc_gemm_tma" -s 40 -c 12 -o $OUT/c2_gemm_full $B --config c2 > /dev/null 2>&1
ls -la $OUT
