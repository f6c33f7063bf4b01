#!/bin/bash
# One profiling pass for a round (run on the GPU box): ncu --set full of the TC
# scan + refine on the bench's index shape, and the launch list of bench.py.
#   tools/prof_round.sh <tag>
tag=${1:-r01}
bash tools/ncu_tc.sh $tag
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$tag.csv python bench.py --steps 3 --warmup 3 --no-latency \
  --no-cpu-baseline > gpurun_out/bench_ncu_$tag.log 2>&1
echo "launch list rc=$?"
