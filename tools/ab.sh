#!/bin/bash
# A/B benchmark of prebuilt libraries: tools/ab.sh libA.so libB.so [rounds]
R=${3:-3}
for r in $(seq $R); do
  for L in "$1" "$2"; do
    QJL_LIB=$L python bench.py --no-cpu-baseline --no-prefill --steps 300 2>/dev/null | python -c "import json,sys;r=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$(basename $L)', round(r['roofline']['achieved']), round(r['value']), r['clocks']['sm_mhz'])"
  done
done
