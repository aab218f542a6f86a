mkdir -p gpurun_out/vbt
for so in abv/*.so; do
  cp $so paper_2511_03909_b200/libwect.so
  n=$(basename $so .so)
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_vbins -s 4 -c 6 --csv python bench.py --config 3 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/vbt/$n.csv 2>/dev/null
done
