#!/bin/bash
# The latency path on the north-star index (10M x 128, C 4096, nprobe 12): a
# 10-query request (the executor's max_search_batch) repeated; the launch list
# with per-launch time + DRAM bytes of every kernel, and a full-set capture of
# one late request's scan kernels.   tools/ncu_lat.sh <tag>
tag=${1:-r02}
mkdir -p gpurun_out
export PROF_NBASE=10000000 PROF_NLIST=4096 PROF_COMPS=256 PROF_TRAIN=262144 PROF_NPROBE=12 PROF_NQ=10 PROF_REPS=40 PROF_QOFF=${PROF_QOFF:-1}
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_lat_$tag.csv python tools/prof_scan.py > gpurun_out/ncu_lat_launch_$tag.log 2>&1
echo "ncu lat launches rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
  -k "regex:scan_vm_kernel|scan_tc_kernel" -s 60 -c 3 -o gpurun_out/prof_lat_$tag \
  python tools/prof_scan.py > gpurun_out/ncu_lat_$tag.log 2>&1
echo "ncu lat full rc=$?"
