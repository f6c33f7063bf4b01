#!/bin/bash
# ncu capture of the CUDA-core exact scan (IP / D > 128 / k > 32 shapes):
#   PROF_D=768 PROF_METRIC=1 PROF_NLIST=4096 PROF_NBASE=2000000 tools/ncu_cuda.sh <tag>
tag=${1:-r01}
PROF_REPS=2 timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k "regex:scan_kernel<.*\(bool\)0>" -s 1 -c 1 -o gpurun_out/prof_cuda_$tag \
  python tools/prof_scan.py > gpurun_out/ncu_cuda_$tag.log 2>&1
echo "ncu cuda rc=$?"
tail -3 gpurun_out/ncu_cuda_$tag.log
