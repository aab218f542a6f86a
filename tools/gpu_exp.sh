# A/B timing of experimental library builds: tools/exp_libwect_<e>.so
for e in ${EXPS:-0 1 2}; do
  if [ "$e" != "0" ]; then export WECT_LIBWECT_OVERRIDE=$PWD/tools/exp_libwect_$e.so; else unset WECT_LIBWECT_OVERRIDE; fi
  r=$(timeout 300 python bench.py --no-cpu --no-e2e ${BENCH_ARGS} 2>&1 | tail -1)
  echo "exp $e: $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("kernel_ms", round(d["roofline"]["kernel_ms"],4), "step_ms", round(d["ms_per_step"],4))' 2>&1)"
done
