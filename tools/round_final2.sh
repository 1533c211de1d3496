#!/bin/bash
# Final pass of the round (run on the GPU box, code as committed): the GPU test
# suite, smoke, every config's bench line, the reference arm and the C2 launch
# list of the timed mode. Usage: bash tools/round_final2.sh <tag>
TAG=${1:-r02o}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/gpu_tests.log
bash tools/round_final.sh $TAG
