#!/bin/bash
# compute-sanitizer passes over the GPU parity tests (run on the GPU box):
#   tools/sanitize.sh <tag>   -> gpurun_out/san_<tool>_<tag>.log
# memcheck over the TC / parity / oracle-direct tests; racecheck and synccheck
# (shared-memory hazards, barrier misuse) over a smaller subset.  racecheck
# models __syncthreads / bar.sync but not mbarrier ordering, so it is pointed at
# the kernels whose shared-memory hand-offs use named barriers (the list scan's
# math warps, the refine, the seed and sample kernels); the CUDA-core scan's
# mbarrier-ordered item ring reports false WAR hazards (profiles/r02_sanitizer.md).
tag=${1:-r02}
mkdir -p gpurun_out
SAN="compute-sanitizer --print-limit 50 --error-exitcode 3"
timeout -s KILL 1500 $SAN --tool memcheck --leak-check no python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_oracle_direct.py -m gpu -x -q -p no:cacheprovider \
  -k "not scale and not cfg5 and not unmodified" > gpurun_out/san_memcheck_$tag.log 2>&1
echo "memcheck rc=$?"
timeout -s KILL 1200 $SAN --tool racecheck --racecheck-report hazard --kernel-name kns=scan_vm_kernel \
  --kernel-name kns=refine_kernel --kernel-name kns=vm_seed --kernel-name kns=sample_ \
  python -m pytest tests/test_gpu_tc.py -m gpu -x -q -p no:cacheprovider \
  -k "tc_equals_exact_and_oracle and (32-16 or 8-6) or seeded_batches and 8-6 or seed_samples" > gpurun_out/san_racecheck_$tag.log 2>&1
echo "racecheck rc=$?"
timeout -s KILL 900 $SAN --tool synccheck python -m pytest tests/test_gpu_tc.py -m gpu -x -q -p no:cacheprovider \
  -k "tc_equals_exact_and_oracle and (32-16 or 8-6) or seeded_batches and 8-6 or seed_samples" > gpurun_out/san_synccheck_$tag.log 2>&1
echo "synccheck rc=$?"
# analysis mode: every distinct (write site, read site) pair once, no backtraces
timeout -s KILL 900 compute-sanitizer --tool racecheck --racecheck-report analysis --show-backtrace no --print-limit 200 \
  --kernel-name kns=scan_vm_kernel --kernel-name kns=refine_kernel --kernel-name kns=vm_seed --kernel-name kns=sample_ \
  python -m pytest tests/test_gpu_tc.py -m gpu -x -q -p no:cacheprovider \
  -k "tc_equals_exact_and_oracle and 8-6 or seed_samples" > gpurun_out/san_raceanalysis_$tag.log 2>&1
echo "racecheck analysis rc=$?"
for f in gpurun_out/san_*_$tag.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" $f | tail -4; done
