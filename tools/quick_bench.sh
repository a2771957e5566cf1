# one short bench; prints value / kernel_ms / roofline frac
python bench.py --no-cpu-baseline --no-prefill --steps ${1:-200} ${@:2} > gpurun_out/qb.log 2>&1
grep '^{' gpurun_out/qb.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value']), 'kernel_us', round(d['roofline']['kernel_ms']*1e3,1), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']))"
