# Round profile set: bench lines + launch list + ncu --set full of each dominant kernel.
set -x
mkdir -p gpurun_out/prof
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/prof/smi.txt
timeout 600 python bench.py > gpurun_out/prof/bench_cfg1.json 2> gpurun_out/prof/bench_cfg1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu > gpurun_out/prof/bench_torchrun1.json 2> gpurun_out/prof/bench_torchrun1.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/prof/launches_cfg1.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
# kernel : bench --config : launches to skip : traffic.json key : extra bench args
for spec in "k_sweep2d:1:2:cfg1:" "k_grid_hist:2:2:cfg2:" "k_cells_vb:3:2:cfg3:" "k_vbins:3:2:cfg3_vbins:" \
            "k_stream:ecfx:2:cfgecfx:" "k_stream:3:2:cfg3_D1:--D 1"; do
  IFS=: read k c s key extra <<< "$spec"
  tag=${key}_$k
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$k\$|$k<" -s $s -c 1 -o /tmp/full_$tag python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --config $c $extra > gpurun_out/prof/full_$tag.log 2>&1
  python tools/ncu_report.py /tmp/full_$tag.ncu-rep gpurun_out/prof/r_$tag.md $key > /dev/null 2>&1
  ncu -i /tmp/full_$tag.ncu-rep --page source --csv --print-source=sass > gpurun_out/prof/src_$tag.csv 2>/dev/null
  gzip -f gpurun_out/prof/src_$tag.csv
done
for c in 0 2 3 4 ecfx; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/prof/bench_cfg$c.json 2> gpurun_out/prof/bench_cfg$c.err; done
for d in 1 4 16 64 256 1024; do timeout 900 python bench.py --config 3 --D $d --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/prof/bench_dsweep_D$d.json 2>/dev/null; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/prof/bench_ref_cfg1.json 2>&1
ls -la gpurun_out/prof
