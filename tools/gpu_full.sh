# full GPU suite + smoke + default bench line
set -x
mkdir -p gpurun_out/full
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/full/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/full/bench_default.json 2> gpurun_out/full/bench_default.err
cat gpurun_out/full/pytest_gpu.txt gpurun_out/full/smoke.txt
