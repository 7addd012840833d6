#!/bin/bash
# Round-2 profile evidence, run on the GPU box from the repo root:
#   1. the driver's bench command plain (must exit 0), then its ncu launch list
#      (gpu__time_duration of the first 400 kernels, cold/serialised)
#   2. per-launch DRAM traffic of each config's default plan (ncu
#      --cache-control none, 10 launches of bench.py's timed graph)
#   3. ncu --set full captures of the c5a / c2 / c3 K1 and c4 K3g kernels,
#      exported as details / raw CSV (the .ncu-rep files stay in /tmp)
#   4. traffic.json (what bench.py reports as roofline.traffic)
cd "$(dirname "$0")/.."
O=gpurun_out/r2
mkdir -p $O
python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_plain.out 2> $O/bench_plain.err
echo "bench plain rc=$?" >> $O/status.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_bench.csv python bench.py --gpus 1 --steps 20 --warmup 5 \
  > $O/bench_ncu.log 2>&1
echo "launch list rc=$?" >> $O/status.txt
for c in c1 c2 c3 c5a c4 c5b; do
  steps=40; [ $c = c4 ] && steps=20; [ $c = c5b ] && steps=14
  timeout 900 ncu --cache-control none --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:'k1_rows|k1m_rows|k3_|k_seg|k4_' -s 10 -c 10 --csv --log-file $O/traffic_$c.csv \
    python bench.py --config $c --extra '' --steps $steps --warmup 3 --no-cpu-baseline \
    --no-parity --e2e-steps 1 --iso-reps 2 > $O/tncu_$c.log 2>&1
  echo "traffic $c rc=$?" >> $O/status.txt
done
full() {  # name config kernel-regex skip reps
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 \
    -o /tmp/prof_$1 python scripts/profile_target.py --config $2 --reps $5 > $O/full_$1.log 2>&1
  echo "full $1 rc=$?" >> $O/status.txt
  ncu -i /tmp/prof_$1.ncu-rep --page details --csv > $O/$1_details.csv 2>&1
  ncu -i /tmp/prof_$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>&1
}
full c5a_k1 c5a k1_rows 2 3
full c2_k1 c2 k1_rows 5 8
full c3_k1 c3 k1_rows 5 8
full c4_k3g c4 k3_gres 1 2
python scripts/traffic_json.py $O $O/traffic.json >> $O/status.txt 2>&1
du -sh $O >> $O/status.txt
