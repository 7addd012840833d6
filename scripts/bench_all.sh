#!/bin/bash
# Run bench.py on every BASELINE config (1 GPU) -> gpurun_out/bench_<cfg>.json
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in "c1 20000" "c2 20000" "c3 20000" "c4 2000" "c5a 400" "c5b 200"; do
  set -- $spec
  timeout 900 python bench.py --config $1 --steps $2 --warmup 20 --no-cpu-baseline --e2e-steps 10 \
    > gpurun_out/bench_$1.json 2> gpurun_out/bench_$1.err
  echo "$1 rc=$?" >> gpurun_out/bench_all.status
done
