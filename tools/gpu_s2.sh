set -x
mkdir -p gpurun_out/s2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/s2/smi.txt
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/s2/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2/smoke.txt 2>&1
for c in 1 0 2 3 4 ecfx; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/s2/bench_cfg$c.json 2> gpurun_out/s2/bench_cfg$c.err; done
tail -3 gpurun_out/s2/pytest_gpu.txt
