#!/bin/bash
# ncu capture of the tensor-core scan + refine (run on the GPU box): tools/ncu_tc.sh <tag>
tag=${1:-r01}
PROF_REPS=2 timeout -s KILL 600 ncu --set full --clock-control none --import-source on \
  -k "regex:scan_tc_kernel|refine_kernel" -s 2 -c 2 -o gpurun_out/prof_tc_$tag \
  python tools/prof_scan.py > gpurun_out/ncu_tc_$tag.log 2>&1
echo "ncu tc rc=$?"
tail -2 gpurun_out/ncu_tc_$tag.log
