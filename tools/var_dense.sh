export PROF_NBASE=1600000 PROF_NLIST=2048 PROF_NPROBE=64 PROF_K=100 PROF_REPS=4
for v in paper_2408_02937_b200/libbivf_gpu.so var/libbivf_r4b6.so var/libbivf_r2b1.so var/libbivf_r2b6.so var/libbivf_r1b1.so var/libbivf_r1b6.so; do
  echo "== $v"; BIVF_LIB=$PWD/$v timeout 300 python tools/prof_scan.py 2>&1 | tail -2
done
