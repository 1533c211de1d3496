#!/bin/bash
# Final measurement pass of a round (run on the GPU box): smoke, every config's
# bench line, the reference arm, and the C2 launch list of the timed mode.
# Usage: bash tools/round_final.sh <tag>
TAG=${1:-r02f}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
timeout 900 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
for c in c1 c3 c4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 900 python bench.py --config c5 --steps 100 --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err
timeout 600 python bench.py --impl reference > $OUT/ref_c2.json 2> $OUT/ref_c2.err
# launch list of the timed mode (resident plans replayed as graphs): ncu
# profiles each graph kernel node; cold-cache and serialised, compare shares
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --graph-profiling node -s 800 -c 240 --csv --log-file $OUT/c2_launches_graph.csv \
  python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-extras --profile-steps 1 > /dev/null 2>&1
ls -la $OUT
