set -x
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "ecf or stream or degenerate or out_of_range or small_D" 2>&1 | tail -15
for i in 1 2; do timeout 600 python bench.py --config ecfx --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ecfx', d['value'], d['ms_per_step'], r['kernel_ms'], r['frac'], d['clocks'])"; done
WECT_DISABLE_VB1=1 timeout 600 python bench.py --config ecfx --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ecfx-kstream', d['value'], d['ms_per_step'], r['kernel_ms'], r['frac'])"
