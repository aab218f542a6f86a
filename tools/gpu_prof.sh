# ncu full capture of one kernel: KREGEX, plus bench args
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_sweep2d} -s ${SKIP:-2} -c 1 -o gpurun_out/${OUT:-prof} python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu ${BENCH_ARGS} > gpurun_out/${OUT:-prof}.log 2>&1
tail -2 gpurun_out/${OUT:-prof}.log
