#!/bin/bash
# Steady-state per-launch DRAM traffic of the default plan for each config
# (ncu --cache-control none; bench loop), plus full captures of c2 and c4.
cd "$(dirname "$0")/.."
for c in c1 c2 c3 c5a c4 c5b; do
  steps=300; [ $c = c4 ] && steps=20; [ $c = c5a ] && steps=20; [ $c = c5b ] && steps=14
  timeout 300 python bench.py --config $c --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/tplain_$c.log 2>&1 || continue
  timeout 600 ncu --cache-control none --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:'k1_rows|k3_|k_seg|k4_' -s 10 -c 10 --csv --log-file gpurun_out/traffic_$c.csv \
    python bench.py --config $c --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/tncu_$c.log 2>&1
done
python scripts/profile_target.py --config c2 --reps 8 > gpurun_out/pt_c2f.log 2>&1 && \
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k1_rows -s 5 -c 1 \
    -o gpurun_out/prof_c2_final python scripts/profile_target.py --config c2 --reps 8 > /dev/null 2>&1
python scripts/profile_target.py --config c4 --reps 2 > gpurun_out/pt_c4f.log 2>&1 && \
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k3_gres -s 1 -c 1 \
    -o gpurun_out/prof_c4_gres python scripts/profile_target.py --config c4 --reps 2 > /dev/null 2>&1
python scripts/traffic_json.py gpurun_out gpurun_out/traffic.json
ls gpurun_out
