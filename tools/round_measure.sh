#!/bin/bash
# One measurement pass (on the GPU box): bench lines for every config, the
# reference arm, and the profile of the default config.
# Usage: bash tools/round_measure.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out
nproc > gpurun_out/${TAG}_host.txt; lscpu | grep "Model name" >> gpurun_out/${TAG}_host.txt
timeout 600 python bench.py > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_ref_c2.json 2> gpurun_out/${TAG}_ref_c2.err
for c in c1 c3 c4; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
timeout 600 python bench.py --config c5 --steps 100 --no-cpu-baseline > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
timeout 900 bash tools/profile_run.sh ${TAG} c2
