# image-ECF loop: GPU parity + bench lines
set -x
timeout 900 python -m pytest tests/test_ecf_images_gpu.py -q -x 2>&1 | tail -15
for c in ecfimg ecfimg1k; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --cpu-budget 5 2>&1 | tail -1 > gpurun_out/bench_$c.json; python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); r=d['roofline']; print('$c', d['value'], d['ms_per_step'], r['kernel_ms'], r['bound'], r['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"; done
