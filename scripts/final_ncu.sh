# steady-state traffic per config + full ncu captures of the c2 (K1) and c4 (K3g) kernels,
# reports kept in /tmp (too large for gpurun_out), exported as CSV
mkdir -p gpurun_out
for c in c1 c2 c3 c5a c4 c5b; do
  steps=300; [ $c = c4 ] && steps=20; [ $c = c5a ] && steps=20; [ $c = c5b ] && steps=14
  timeout 600 ncu --cache-control none --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:'k1_rows|k3_|k_seg|k4_' -s 10 -c 10 --csv --log-file gpurun_out/traffic_$c.csv \
    python bench.py --config $c --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 1 > /tmp/tncu_$c.log 2>&1
  echo "traffic $c rc=$?" >> gpurun_out/ncu_status.txt
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k1_rows -s 5 -c 1 \
  -o /tmp/prof_c2 python scripts/profile_target.py --config c2 --reps 8 > /tmp/p2.log 2>&1
echo "full c2 rc=$?" >> gpurun_out/ncu_status.txt
ncu -i /tmp/prof_c2.ncu-rep --page details --csv > gpurun_out/c2_k1_details.csv 2>&1
ncu -i /tmp/prof_c2.ncu-rep --page raw --csv > gpurun_out/c2_k1_raw.csv 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k3_gres -s 1 -c 1 \
  -o /tmp/prof_c4 python scripts/profile_target.py --config c4 --reps 2 > /tmp/p4.log 2>&1
echo "full c4 rc=$?" >> gpurun_out/ncu_status.txt
ncu -i /tmp/prof_c4.ncu-rep --page details --csv > gpurun_out/c4_k3g_details.csv 2>&1
python scripts/traffic_json.py gpurun_out gpurun_out/traffic.json >> gpurun_out/ncu_status.txt 2>&1
du -sh gpurun_out >> gpurun_out/ncu_status.txt
