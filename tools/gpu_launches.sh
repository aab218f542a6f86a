# ncu launch list (gpu__time_duration per launch) of one bench config: CONFIG, STEPS
mkdir -p gpurun_out/ll
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll/launches_cfg${CONFIG:-1}.csv \
  python bench.py --config ${CONFIG:-1} --steps ${STEPS:-1} --warmup ${WARMUP:-3} --no-e2e --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv, collections, os
c = os.environ.get("CONFIG", "1")
rows = [r for r in csv.reader(open(f"gpurun_out/ll/launches_cfg{c}.csv")) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
t = collections.defaultdict(float); n = collections.Counter()
for r in rows[1:]:
    k = r[ki].split("(")[0].split("<")[0]
    t[k] += float(r[vi].replace(",", "")); n[k] += 1
tot = sum(t.values())
for k, v in sorted(t.items(), key=lambda x: -x[1])[:15]:
    print(f"{k:40s} {n[k]:5d} launches {v/1e6:9.3f} ms {100*v/tot:5.1f}%")
PY
