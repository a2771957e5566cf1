#!/bin/bash
# A/B/n benchmark of prebuilt libraries: tools/ab_multi.sh ROUNDS lib1.so lib2.so ...
R=$1; shift
for r in $(seq $R); do
  for L in "$@"; do
    QJL_LIB=$L python bench.py --no-cpu-baseline --no-prefill --steps 300 2>/dev/null | python -c "import json,sys;r=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$(basename $L)', 'kernel_GBs', round(r['roofline']['achieved']), 'step_GBs', round(r['value']), 'us', round(r['roofline']['kernel_ms']*1e3,1), r['clocks']['sm_mhz'])"
  done
done
