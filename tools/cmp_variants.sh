for v in libbivf_gpu.so libbivf_gpu_prof.so; do
  export BIVF_LIB=$PWD/paper_2408_02937_b200/$v
  echo "== $v"
  timeout 300 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
  timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1
  tail -1 gpurun_out/bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['phase_ms'], d['latency']['search_live_inserts_ms']['p99_ms'])"
done
