# round evidence: the GPU test suite, every bench line, launch lists of the default / ECF-X /
# cfg4 commands, ncu --set full of the dominant kernels (summarised into gpurun_out/ev/ by
# tools/ncu_report.py; raw and source pages kept as csv)
mkdir -p gpurun_out/ev
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ev/build.log 2>&1 || { tail -30 gpurun_out/ev/build.log; exit 1; }
if [ -z "$NO_TESTS" ]; then
  timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/ev/pytest_gpu.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/ev/smoke.txt 2>&1
fi
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw --format=csv > gpurun_out/ev/smi.txt
timeout 900 python bench.py > gpurun_out/ev/bench_cfg1.json 2> gpurun_out/ev/bench_cfg1.err
for c in ${CONFIGS:-0 2 3 4 ecfx ecfimg ecfimg1k freud bwd3 bwd4}; do
  timeout 900 python bench.py --config $c --steps 10 > gpurun_out/ev/bench_cfg$c.json 2> gpurun_out/ev/bench_cfg$c.err
done
WECT_IMAGES_MMA=1 timeout 600 python bench.py --steps 10 > gpurun_out/ev/bench_cfg1_mma.json 2> gpurun_out/ev/bench_cfg1_mma.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev/bench_ref_cfg1.json 2>/dev/null
for spec in "1:2:3" "ecfx:2:3" "3:1:1"; do
  IFS=: read c s w <<< "$spec"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_cfg$c.csv \
    python bench.py --config $c --steps $s --warmup $w --no-e2e --no-cpu > /dev/null 2>&1
done
for spec in "1:k_sweep2d:3" "ecfx:k_stream:3" "2:k_grid_hist:3" "3:k_cells_vb:8" "freud:k_sweep2d:3" "4:k_cells_vb:4"; do
  IFS=: read c k s <<< "$spec"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -o gpurun_out/ev/full_${c}_${k} \
    python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ev/full_${c}_${k}.log 2>&1
  python tools/ncu_report.py gpurun_out/ev/full_${c}_${k}.ncu-rep gpurun_out/ev/r02_${k}_cfg${c}.md cfg$c > /dev/null 2>&1
  ncu -i gpurun_out/ev/full_${c}_${k}.ncu-rep --page raw --csv > gpurun_out/ev/r02_${k}_cfg${c}.raw.csv 2>/dev/null
  rm -f gpurun_out/ev/full_${c}_${k}.ncu-rep
done
ls gpurun_out/ev
