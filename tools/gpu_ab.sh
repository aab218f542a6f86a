# A/B timing of prebuilt libwect variants (abv/*.so) on one box: kernel ms of the dominant
# kernel for each config in $CONFIGS (timing only; variants may compute wrong results)
# ($EXTRA: more bench arguments, e.g. "--D 8")
mkdir -p gpurun_out/ab
cp paper_2511_03909_b200/libwect.so /tmp/libwect_orig.so
for rep in 1 2; do
for so in abv/*.so; do
  cp $so paper_2511_03909_b200/libwect.so
  for c in ${CONFIGS:-1}; do
    timeout 300 python bench.py --config $c $EXTRA --no-cpu --no-e2e --steps 20 2>/dev/null | tail -1 > gpurun_out/ab/x.json
    python -c "import json; d=json.load(open('gpurun_out/ab/x.json')); r=d['roofline']; print('$so', 'cfg $c', 'kernel_ms %.4f' % r.get('kernel_ms'), 'step_ms %.4f' % d['ms_per_step'])" 2>/dev/null || echo "$so cfg $c failed"
  done
done
done
cp /tmp/libwect_orig.so paper_2511_03909_b200/libwect.so
