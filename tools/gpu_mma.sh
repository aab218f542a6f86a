# tensor-core image path: parity tests + timing beside the sweep (+ optional ncu)
mkdir -p gpurun_out/mma
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/mma/build.log 2>&1 || { tail -30 gpurun_out/mma/build.log; exit 1; }
timeout 300 python -m pytest tests/test_mma_gpu.py -q -x ${MMA_K:+-k "$MMA_K"} 2>&1 | tail -15 | tee gpurun_out/mma/pytest.txt
for e in 0 1; do
  WECT_IMAGES_MMA=$e timeout 300 python bench.py --config 1 --no-cpu --no-e2e --steps 20 > gpurun_out/mma/bench_$e.json 2> gpurun_out/mma/bench_$e.err
  python -c "import json; d=json.load(open('gpurun_out/mma/bench_$e.json')); r=d['roofline']; print('mma=$e', 'value', d['value'], 'step_ms %.4f' % d['ms_per_step'], 'kernel', r.get('kernel'), 'kernel_ms', r.get('kernel_ms'), 'frac', r.get('frac'))" || tail -5 gpurun_out/mma/bench_$e.err
done
if [ -n "$MMA_NCU" ]; then
  WECT_IMAGES_MMA=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_mma2d -s 2 -c 1 -o gpurun_out/mma/full_mma \
    python bench.py --config 1 --steps 2 --warmup 2 --no-e2e --no-cpu > gpurun_out/mma/ncu.log 2>&1
  python tools/ncu_report.py gpurun_out/mma/full_mma.ncu-rep gpurun_out/mma/r02_k_mma2d_cfg1.md cfg1 > /dev/null 2>&1
  ncu -i gpurun_out/mma/full_mma.ncu-rep --page source --csv > gpurun_out/mma/r02_k_mma2d_cfg1.src.csv 2>/dev/null
  ncu -i gpurun_out/mma/full_mma.ncu-rep --page raw --csv > gpurun_out/mma/r02_k_mma2d_cfg1.raw.csv 2>/dev/null
  rm -f gpurun_out/mma/full_mma.ncu-rep
fi
