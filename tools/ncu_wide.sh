#!/bin/bash
# ncu capture of the inner-product wide mode (run on the GPU box): tools/ncu_wide.sh <tag>
# 2M x 768 normalised synthetic vectors, nlist 1024, IP; one search skipped (5
# launches: TC IP quantizer scan + refine, seeding scan, full scan, refine), the
# second search's 5 captured.
tag=${1:-r01}
PROF_NBASE=2000000 PROF_D=768 PROF_METRIC=1 PROF_NLIST=1024 PROF_REPS=2 timeout -s KILL 900 \
  ncu --set full --clock-control none --import-source on \
  -k "regex:scan_tc_kernel|refine_kernel" -s 5 -c 5 -o gpurun_out/prof_wide_$tag \
  python tools/prof_scan.py > gpurun_out/ncu_wide_$tag.log 2>&1
echo "ncu wide rc=$?"
tail -2 gpurun_out/ncu_wide_$tag.log
