# one ncu --set full capture of kernel KREGEX for bench config CFG (plus bench line first)
mkdir -p gpurun_out/n1
timeout 300 python bench.py --config ${CFG:-ecfx} --no-cpu --no-e2e --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['workload'], d['value'], 'ms', d['ms_per_step'], 'kernel_ms', r.get('kernel_ms'), 'frac', r['frac'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_stream} -s ${SKIP:-3} -c 1 -o gpurun_out/n1/${OUT:-k} python bench.py --config ${CFG:-ecfx} --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/n1/${OUT:-k}.log 2>&1
tail -1 gpurun_out/n1/${OUT:-k}.log
