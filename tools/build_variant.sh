#!/bin/bash
# Build a variant of the library with extra -D flags on scan_tc.cu:
#   tools/build_variant.sh <name> -DFOO=1 ...  ->  var/libbivf_<name>.so
# Use it through BIVF_LIB=$PWD/var/libbivf_<name>.so.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
python -c "import sys; sys.path.insert(0,'.'); from paper_2408_02937_b200 import build as b; b.build(verbose=False)"
mkdir -p var build/var
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -ffp-contract=off -I paper_2408_02937_b200/csrc -I include "$@" \
  -c paper_2408_02937_b200/csrc/scan_tc.cu -o build/var/scan_tc_$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o var/libbivf_$name.so $(ls build/bivf/*.o | grep -v scan_tc) build/var/scan_tc_$name.o -lpthread -lgomp -ldl
