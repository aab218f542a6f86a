# round evidence: every bench line, the default command's launch list, ncu --set full of the
# dominant kernels (summarised locally by tools/ncu_report.py into profiles/)
mkdir -p gpurun_out/ev
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw --format=csv > gpurun_out/ev/smi.txt
timeout 900 python bench.py > gpurun_out/ev/bench_cfg1.json 2> gpurun_out/ev/bench_cfg1.err
for c in ${CONFIGS:-0 2 3 4 ecfx ecfimg ecfimg1k freud bwd3 bwd4}; do
  timeout 900 python bench.py --config $c --steps 10 > gpurun_out/ev/bench_cfg$c.json 2> gpurun_out/ev/bench_cfg$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev/bench_ref_cfg1.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_cfg1.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_ecfx.csv \
  python bench.py --config ecfx --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
for spec in "1:k_sweep2d:3" "ecfx:k_stream:3" "2:k_grid_hist:3" "3:k_cells_vb:8" "freud:k_sweep2d:3"; do
  IFS=: read c k s <<< "$spec"
  timeout 900 ncu --set full --clock-control none -k regex:$k -s $s -c 1 -o gpurun_out/ev/full_${c}_${k} \
    python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ev/full_${c}_${k}.log 2>&1
  # summarise here (a full report is ~30 MB: too big to bring back), keep the summary + raw csv
  python tools/ncu_report.py gpurun_out/ev/full_${c}_${k}.ncu-rep gpurun_out/ev/r02_${k}_cfg${c}.md cfg$c > /dev/null 2>&1
  ncu -i gpurun_out/ev/full_${c}_${k}.ncu-rep --page raw --csv > gpurun_out/ev/r02_${k}_cfg${c}.raw.csv 2>/dev/null
  rm -f gpurun_out/ev/full_${c}_${k}.ncu-rep
done
ls gpurun_out/ev
