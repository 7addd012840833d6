#!/bin/bash
# long-row shapes: planner default vs K3c (gres off) vs K3g (forced) vs split
cd "$(dirname "$0")/.."
for shp in 4096x16384 2048x32768 2048x65536 1024x131072 512x262144 256x524288 256x1048576 64x2097152; do
  timeout 200 python scripts/sweep.py --shape $shp --only-resident --reps 40 --gres-ps 0 2>&1 | grep -v "sk_copy\|Traceback\|^  " 
done
