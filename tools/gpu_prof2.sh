# round-1 (session 2) profile set: ncu --set full of the new / changed kernels + sources
set -x
mkdir -p gpurun_out/p2
for spec in "k_stream:ecfx:2:cfgecfx" "k_ecf_img2d_w4:ecfimg:2:cfgecfimg" "k_ecf_img_hist:ecfimg1k:2:cfgecfimg1k" "k_grad_cells:bwd4:4:cfgbwd4" "k_sweep2d:1:2:cfg1"; do
  IFS=: read k c s key <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$k\$|$k<" -s $s -c 1 -o gpurun_out/p2/full_$key python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --config $c > gpurun_out/p2/full_$key.log 2>&1
  ncu -i gpurun_out/p2/full_$key.ncu-rep --page source --csv --print-source=sass > gpurun_out/p2/src_$key.csv 2>/dev/null
  python tools/ncu_report.py gpurun_out/p2/full_$key.ncu-rep gpurun_out/p2/r01_${k}_$key.md $key > /dev/null 2>&1
  gzip -f gpurun_out/p2/src_$key.csv
  mv gpurun_out/p2/full_$key.ncu-rep /tmp/
done
cp profiles/traffic.json gpurun_out/p2/traffic.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p2/launches_cfg1.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p2/launches_ecfimg.csv python bench.py --config ecfimg --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ls -la gpurun_out/p2
