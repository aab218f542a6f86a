# sweep iteration loop: image parity subset + cfg2/cfg1/freud bench lines (+ optional ncu of k_sweep2d)
mkdir -p gpurun_out/sw
timeout 900 python -m pytest tests -m gpu -q -x -k "${PYTEST_K:-images or cfg1 or cfg2 or freud or graph}" 2>&1 | tail -8
for c in ${CONFIGS:-1}; do
  timeout 300 python bench.py --config $c --no-cpu --no-e2e --steps 20 2>gpurun_out/sw/b$c.err | tail -1 > gpurun_out/sw/b$c.json
  python -c "import json,sys; d=json.load(open('gpurun_out/sw/b$c.json')); r=d['roofline']; print('cfg $c', d['value'], d['unit'], 'ms', d['ms_per_step'], 'kernel_ms', r.get('kernel_ms'), 'frac', r['frac'], d['clocks'].get('sm_mhz'))" || tail -3 gpurun_out/sw/b$c.err
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep2d -s 2 -c 1 -o gpurun_out/sw/sweep python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/sw/ncu.log 2>&1
  tail -2 gpurun_out/sw/ncu.log
fi
