#!/bin/bash
# ncu capture of the tensor-core scan + refine (run on the GPU box): tools/ncu_tc.sh <tag>
# prof_scan.py builds the cfg2 index on the CUDA-core path, then searches; the
# first search's 5 launches (TC quantizer + its selection, the two-phase TC list
# scan, refine) are skipped, the second search's 5 captured.
tag=${1:-r01}
PROF_REPS=2 timeout -s KILL 600 ncu --set full --clock-control none --import-source on \
  -k "regex:scan_tc_kernel|refine_kernel|dense_" -s 5 -c 5 -o gpurun_out/prof_tc_$tag \
  python tools/prof_scan.py > gpurun_out/ncu_tc_$tag.log 2>&1
echo "ncu tc rc=$?"
tail -2 gpurun_out/ncu_tc_$tag.log
