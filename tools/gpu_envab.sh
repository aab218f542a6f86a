# A/B of an environment switch on one box: kernel ms of the dominant kernel for $CONFIGS with
# $ENVVAR unset / set to 1, alternated $REPS times (timing only)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
[ -n "$PYTEST_K" ] && timeout 900 python -m pytest tests -m gpu -q -x -k "$PYTEST_K" 2>&1 | tail -3
for rep in $(seq ${REPS:-2}); do
  for v in "" 1; do
    for c in ${CONFIGS:-1}; do
      if [ -z "$v" ]; then pre="env -u $ENVVAR"; else pre="env $ENVVAR=$v"; fi
      $pre timeout 300 python bench.py --config $c --no-cpu --no-e2e --steps 20 > /tmp/ab.json 2>/dev/null
      python -c "import json; d=json.load(open('/tmp/ab.json')); print('$ENVVAR=${v:-unset}', 'cfg $c', 'kernel_ms %.4f' % d['roofline']['kernel_ms'], 'step_ms %.4f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'])"
    done
  done
done
