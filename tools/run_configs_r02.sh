#!/bin/bash
# Round-2 secondary configs (GPU box): one JSON line per BASELINE config other
# than the headline, clocks sampled in the timed region, cpu_baseline + parity on
# a bounded sample.   tools/run_configs_r02.sh [configs...]
mkdir -p gpurun_out/configs_r02
cfgs=${@:-cfg1 cfg3 cfg4s cfg5s cfg5}
for c in $cfgs; do
  extra="--cpu-baseline"
  [ "$c" = cfg5 ] && extra=""   # the restatement would need the whole 61 GB index on the host: cfg5s carries it
  timeout -s KILL 1500 python tools/bench_configs.py --config $c --steps 10 --warmup 3 $extra \
    > gpurun_out/configs_r02/$c.json 2> gpurun_out/configs_r02/$c.log
  echo "$c rc=$? $(head -c 300 gpurun_out/configs_r02/$c.json)"
done
