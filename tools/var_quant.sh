#!/bin/bash
# Compare library variants (var/*.so) on the quantizer phase: cfg2 proxy (nprobe 32)
# and the cfg4-shard proxy (nprobe 64, k 100).
for v in paper_2408_02937_b200/libbivf_gpu.so var/*.so; do
  echo "== $v"
  BIVF_LIB=$PWD/$v PROF_REPS=4 timeout 300 python tools/prof_scan.py 2>&1 | tail -1
  BIVF_LIB=$PWD/$v PROF_NBASE=1600000 PROF_NLIST=2048 PROF_NPROBE=64 PROF_K=100 PROF_REPS=4 \
    timeout 300 python tools/prof_scan.py 2>&1 | tail -1
done
