#!/bin/bash
# Build libbivf_gpu_prof.so: the library with the scan kernel's per-role cycle
# accounting compiled in (-DBIVF_TC_PROF=1; CTA 0 prints [tc-prof] lines).
# Use it through BIVF_LIB=$PWD/paper_2408_02937_b200/libbivf_gpu_prof.so.
set -e
cd "$(dirname "$0")/.."
python -c "import sys; sys.path.insert(0,'.'); from paper_2408_02937_b200 import build as b; b.build(verbose=False)"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -ffp-contract=off -I paper_2408_02937_b200/csrc -I include -DBIVF_TC_PROF=1 \
  -c paper_2408_02937_b200/csrc/scan_tc.cu -o build/scan_tc_prof.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o paper_2408_02937_b200/libbivf_gpu_prof.so $(ls build/bivf/*.o | grep -v scan_tc) \
  build/scan_tc_prof.o -lpthread -lgomp
