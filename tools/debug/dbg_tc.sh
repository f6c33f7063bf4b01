run() { name=$1; shift; n=$1; shift; f=0; for i in $(seq $n); do timeout 300 python -m pytest -q -p no:cacheprovider "$@" > /tmp/o.txt 2>&1 || { f=$((f+1)); grep -E "^FAILED" /tmp/o.txt | head -3; }; done; echo "== $name: $f of $n failed"; }
Q=tests/test_gpu_parity.py::test_quantizer_exact_at_scale
run A 10 $Q
run ALL 3 tests -m gpu
