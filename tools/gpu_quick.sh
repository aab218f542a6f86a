# quick loop: GPU parity subset + default bench line
set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "${PYTEST_K:-images or cfg1 or cfg2}" 2>&1 | tail -5
timeout 300 python bench.py --no-cpu --no-e2e ${BENCH_ARGS} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'ms',d['ms_per_step'],'kernel_ms',d['roofline']['kernel_ms'],'frac',d['roofline']['frac'], d['clocks'])"
