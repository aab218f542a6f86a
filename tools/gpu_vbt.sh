# per-launch ncu durations of the kernels matching $KRE for each prebuilt abv/*.so on
# bench --config $CFG (A/B of a non-dominant kernel; the last variant stays installed)
mkdir -p gpurun_out/vbt
for so in abv/*.so; do
  cp $so paper_2511_03909_b200/libwect.so
  n=$(basename $so .so)
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:${KRE:-k_vbins} -s ${SKIP:-4} -c ${COUNT:-6} --csv python bench.py --config ${CFG:-3} --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/vbt/$n.csv 2>/dev/null
done
