# per-kernel times of the C2 decode steps (ncu launch list, cold-cache serialised)
timeout 300 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu-baseline --no-prefill --no-extras > gpurun_out/c2plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv -k regex:k_u python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu-baseline --no-prefill --no-extras > /dev/null 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/c2_launches.csv")))
h = None
for r in rows:
    if "Kernel Name" in r:
        h = r; continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        print(d["Kernel Name"][:40], d["Metric Value"])
PY
