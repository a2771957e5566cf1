# m = 512 decode: GPU tests, then C5 points with m = 512 for the shipped library vs $1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for pt in "--batch 16 --n 32768" "--batch 64 --n 32768" "--batch 16 --n 131072" "--batch 4 --n 4096"; do
  for L in $1 paper_2406_03482_b200/libqjl_b200.so; do
    QJL_LIB=$L timeout 300 python bench.py --workload c5 $pt --m-in 512 --steps 30 --warmup 5 --no-cpu-baseline --no-prefill --no-extras 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$(basename $L)', '$pt', 'step_us', round(d['ms_per_step']*1e3,1), 'GB/s', round(d['value']), 'kernel frac', round(d['roofline']['frac'],3))"
  done
done
