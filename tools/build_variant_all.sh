#!/bin/bash
# Build a variant of the whole library (every source) with extra -D flags, for
# flags read outside scan_tc.cu (e.g. -DBIVF_SAMP_S=64):
#   tools/build_variant_all.sh <name> -DFOO=1 ...  ->  var/libbivf_<name>.so
# Use it through BIVF_LIB=$PWD/var/libbivf_<name>.so.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p var build/var_$name
objs=()
for src in scan.cu scan_tc.cu insert.cu maint.cu mirror.cu index.cpp host_algos.cpp executor.cpp capi.cpp group.cpp; do
  x=""; [[ $src == *.cpp ]] && x="-x cu"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
    -Xcompiler -fopenmp -I paper_2408_02937_b200/csrc -I include "$@" $x -c paper_2408_02937_b200/csrc/$src \
    -o build/var_$name/$src.o &
  objs+=(build/var_$name/$src.o)
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o var/libbivf_$name.so "${objs[@]}" -lpthread -lgomp -ldl
echo "built var/libbivf_$name.so"
