#!/bin/bash
# ncu capture of the k > 32 dense path (cfg4 shard proxy: 1.6M x 128 SIFT-like,
# nlist 2048 -> ~780 vectors per list like cfg4's 12.5M/16384, nprobe 64, k 100):
# tools/ncu_dense.sh <tag>.  Timed phases first (no profiler), then the select
# kernel and the dense scan captured on the second search.
tag=${1:-r01}
export PROF_NBASE=1600000 PROF_NLIST=2048 PROF_NPROBE=64 PROF_K=100
  ncu --set full --clock-control none --import-source on \
  -k "regex:dense_.*select" -s 2 -c 2 -o gpurun_out/prof_dsel_$tag \
  python tools/prof_scan.py > gpurun_out/ncu_dsel_$tag.log 2>&1
echo "ncu dense rc=$?"
tail -2 gpurun_out/ncu_dsel_$tag.log
