#!/bin/bash
# Compare library variants (var/libbivf_<name>.so from tools/build_variant.sh) against
# the in-tree library on the k > 32 dense path (cfg4-shard proxy, see ncu_dense.sh).
export PROF_NBASE=1600000 PROF_NLIST=2048 PROF_NPROBE=64 PROF_K=100 PROF_REPS=5
for v in paper_2408_02937_b200/libbivf_gpu.so var/*.so paper_2408_02937_b200/libbivf_gpu.so; do
  echo "== $v"; BIVF_LIB=$PWD/$v timeout 300 python tools/prof_scan.py 2>&1 | tail -2
done
