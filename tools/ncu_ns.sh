#!/bin/bash
# ncu captures on the north-star workload (10M x 128, C 4096, nprobe 12): the
# launch list of one bench run (per-kernel times, cold and serialised) and a
# full-set capture of the second search's kernels (quantizer, seeding scan,
# full scan, refine).  tools/ncu_ns.sh <tag>
tag=${1:-r02}
mkdir -p gpurun_out
export PROF_NBASE=10000000 PROF_NLIST=4096 PROF_COMPS=256 PROF_TRAIN=262144 PROF_NPROBE=12 PROF_REPS=2
timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
  -k "regex:scan_tc_kernel|refine_kernel|dense_" -s 5 -c 5 -o gpurun_out/prof_ns_$tag \
  python tools/prof_scan.py > gpurun_out/ncu_ns_$tag.log 2>&1
echo "ncu full rc=$?"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_ns_$tag.csv python tools/prof_scan.py > gpurun_out/ncu_ns_launch_$tag.log 2>&1
echo "ncu launches rc=$?"
tail -3 gpurun_out/ncu_ns_$tag.log
