#!/bin/bash
# ncu captures of the IVF list-scan kernel (the FLAT instantiation is the quantizer / k-means).
# usage: tools/ncu_scan.sh <tag>   (run on the GPU box; writes gpurun_out/)
tag=${1:-r01}
PROF_REPS=${PROF_REPS:-3} timeout 600 ncu --set full --clock-control none --import-source on \
  --kernel-name-base mangled -k regex:scan_kernelILi1ELi0ELb0 -s 1 -c 1 -o gpurun_out/prof_scan_$tag \
  python tools/prof_scan.py > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu full rc=$?"
tail -2 gpurun_out/ncu_full_$tag.log
