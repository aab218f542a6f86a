# session-2 final profile set: ncu summaries of the kernels changed late + every bench line
set -x
mkdir -p gpurun_out/p4
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/p4/smi.txt
for spec in "k_sweep2d:1:2:cfg1" "k_ecf_img2d_rows:ecfimg1k:2:cfgecfimg1k" "k_grad_cells:bwd3:4:cfgbwd3" "k_grad_cells:bwd4:4:cfgbwd4" "k_sweep2d:freud:2:cfgfreud"; do
  IFS=: read k c s key <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$k\$|$k<" -s $s -c 1 -o /tmp/full_$key python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --config $c > gpurun_out/p4/full_$key.log 2>&1
  python tools/ncu_report.py /tmp/full_$key.ncu-rep gpurun_out/p4/r01_${k}_$key.md $key > /dev/null 2>&1
done
cp profiles/traffic.json gpurun_out/p4/traffic.json
for c in 1 0 2 3 4 ecfx ecfimg ecfimg1k bwd3 bwd4 freud; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --cpu-budget 10 > gpurun_out/p4/bench_$c.json 2> gpurun_out/p4/bench_$c.err; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/p4/bench_ref_cfg1.json 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu > gpurun_out/p4/bench_torchrun1.json 2> gpurun_out/p4/bench_torchrun1.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p4/launches_cfg1.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ls -la gpurun_out/p4
