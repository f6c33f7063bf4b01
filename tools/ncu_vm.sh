#!/bin/bash
# ncu --set full of the vector-major scan on the north-star index (10M x 128,
# C 4096, nprobe 12): the second search's seed, scan and refine launches.
#   tools/ncu_vm.sh <tag>
tag=${1:-r02}
mkdir -p gpurun_out
export PROF_NBASE=10000000 PROF_NLIST=4096 PROF_COMPS=256 PROF_TRAIN=262144 PROF_NPROBE=12 PROF_REPS=2
timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
  -k "regex:scan_vm_kernel|refine_kernel|vm_seed" -s 3 -c 3 -o gpurun_out/prof_vm_$tag \
  python tools/prof_scan.py > gpurun_out/ncu_vm_$tag.log 2>&1
echo "ncu vm rc=$?"
