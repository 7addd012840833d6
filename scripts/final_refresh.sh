rm -f gpurun_out/bench_all.status
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/bench_all.status
timeout 300 python scripts/shard_shapes.py --shapes 8x50257,32x151936,16x262144,64x128256,1024x50257 --points split,split3 > gpurun_out/split2_ab.jsonl 2> gpurun_out/split2_ab.err
bash scripts/bench_all.sh
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "default rc=$?" >> gpurun_out/bench_all.status
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?" >> gpurun_out/bench_all.status
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 200 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?" >> gpurun_out/bench_all.status
du -sh gpurun_out >> gpurun_out/bench_all.status
