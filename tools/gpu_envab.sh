# A/B of env switches on one box: kernel ms of the dominant kernel, config $CONFIGS,
# variants in $VARIANTS ("-" = no env), each as ENV=1
mkdir -p gpurun_out/ab
for rep in 1 2; do
for v in ${VARIANTS:--}; do
  for c in ${CONFIGS:-1}; do
    if [ "$v" = "-" ]; then E=""; else E="$v=1"; fi
    env $E timeout 300 python bench.py --config $c --no-cpu --no-e2e --steps 20 2>/dev/null | tail -1 > gpurun_out/ab/x.json
    python -c "import json; d=json.load(open('gpurun_out/ab/x.json')); r=d['roofline']; print('$v', 'cfg $c', 'kernel_ms %.4f' % r.get('kernel_ms'), 'step_ms %.4f' % d['ms_per_step'])" 2>/dev/null || echo "$v cfg $c failed"
  done
done
done
