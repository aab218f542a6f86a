set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv
timeout 600 python bench.py 2>&1 | tail -3 | tee gpurun_out/bench_cfg1.txt
timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu 2>&1 | tail -3 | tee gpurun_out/bench_cfg2.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_cfg1.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep2d -s 2 -c 1 -o gpurun_out/prof_sweep python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 2>&1 | tail -3 | tee gpurun_out/bench_cfg3.txt
timeout 600 python bench.py --config ecfx --steps 10 --warmup 3 2>&1 | tail -3 | tee gpurun_out/bench_ecfx.txt
