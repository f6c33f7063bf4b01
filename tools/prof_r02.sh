#!/bin/bash
# Round-2 profiling pass (GPU box): ncu --set full of the north-star search
# (quantizer, scan_vm_kernel, refine), the launch list of bench.py, and the
# 10-query latency path.   tools/prof_r02.sh <tag>
tag=${1:-r02}
mkdir -p gpurun_out
export PROF_NBASE=10000000 PROF_NLIST=4096 PROF_COMPS=256 PROF_TRAIN=262144 PROF_NPROBE=12 PROF_REPS=2
timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
  -k "regex:scan_vm_kernel|refine_kernel|scan_tc_kernel|dense_select" -s 4 -c 4 -o gpurun_out/prof_ns_$tag \
  python tools/prof_scan.py > gpurun_out/ncu_ns_$tag.log 2>&1
echo "ncu north-star rc=$?"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$tag.csv python bench.py --steps 3 --warmup 3 --no-latency \
  --no-cpu-baseline > gpurun_out/bench_ncu_$tag.log 2>&1
echo "launch list rc=$?"
bash tools/ncu_lat.sh $tag
