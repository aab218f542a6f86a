set -x
for c in bwd3 bwd4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_$c.json; python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); r=d['roofline']; print('$c', d['value'], d['ms_per_step'], r['kernel_ms'], r['launches_per_step'], r['bound'], r['frac'], d['e2e']['value'], d['cpu_baseline'], d['clocks'])"; done
