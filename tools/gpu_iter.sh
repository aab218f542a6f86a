# iteration loop: build, a GPU test subset ($PYTEST_K), bench lines for $CONFIGS (kernel ms),
# optional ncu --set full of $NCU_SPEC ("config:kernel_regex:skip" items) summarised to gpurun_out/it/
set -x
mkdir -p gpurun_out/it
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/it/build.log 2>&1 || { tail -30 gpurun_out/it/build.log; exit 1; }
if [ -n "$PYTEST_K" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -k "$PYTEST_K" 2>&1 | tail -8 | tee gpurun_out/it/pytest.txt
fi
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv,noheader > gpurun_out/it/smi.txt
for c in ${CONFIGS:-1}; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps ${STEPS:-20} > gpurun_out/it/bench_$c.json 2> gpurun_out/it/bench_$c.err
  python -c "import json; d=json.load(open('gpurun_out/it/bench_$c.json')); r=d['roofline']; print('cfg $c', 'value', d['value'], 'step_ms %.4f' % d['ms_per_step'], 'kernel_ms', r.get('kernel_ms'), 'frac', r.get('frac'), r.get('bound'))" || tail -5 gpurun_out/it/bench_$c.err
done
for spec in $NCU_SPEC; do
  IFS=: read c k s <<< "$spec"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -o gpurun_out/it/full_${c}_${k} \
    python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/it/full_${c}_${k}.log 2>&1
  python tools/ncu_report.py gpurun_out/it/full_${c}_${k}.ncu-rep gpurun_out/it/r02_${k}_cfg${c}.md cfg$c > /dev/null 2>&1
  ncu -i gpurun_out/it/full_${c}_${k}.ncu-rep --page raw --csv > gpurun_out/it/r02_${k}_cfg${c}.raw.csv 2>/dev/null
  ncu -i gpurun_out/it/full_${c}_${k}.ncu-rep --page source --csv > gpurun_out/it/r02_${k}_cfg${c}.src.csv 2>/dev/null
  rm -f gpurun_out/it/full_${c}_${k}.ncu-rep
done
ls gpurun_out/it
