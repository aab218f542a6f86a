# refresh of the remaining profile summaries + every bench line (small outputs only)
set -x
mkdir -p gpurun_out/p3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/p3/smi.txt
for spec in "k_grid_hist:2:2:cfg2::" "k_cells_vb:3:2:cfg3::" "k_vbins:3:2:cfg3_vbins::" "k_stream:3:2:cfg3_D1:--D 1:"; do
  IFS=: read k c s key extra _ <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$k\$|$k<" -s $s -c 1 -o /tmp/full_$key python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --config $c $extra > gpurun_out/p3/full_$key.log 2>&1
  python tools/ncu_report.py /tmp/full_$key.ncu-rep gpurun_out/p3/r01_${k}_$key.md $key > /dev/null 2>&1
done
for c in 1 0 2 3 4 ecfx ecfimg ecfimg1k bwd3 bwd4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --cpu-budget 10 > gpurun_out/p3/bench_$c.json 2> gpurun_out/p3/bench_$c.err; done
for d in 1 2 4 8 16 64 256 1024; do timeout 900 python bench.py --config 3 --D $d --steps 3 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 >> gpurun_out/p3/dsweep_cfg4.jsonl; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/p3/bench_ref_cfg1.json 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu > gpurun_out/p3/bench_torchrun1.json 2> gpurun_out/p3/bench_torchrun1.err
ls -la gpurun_out/p3
