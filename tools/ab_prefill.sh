#!/bin/bash
# A/B of the config-4 prefill (K1) across prebuilt libraries: tools/ab_prefill.sh libA.so libB.so [rounds]
R=${3:-2}
for r in $(seq $R); do
  for L in "$1" "$2"; do
    QJL_LIB=$L python tools/run_prefill.py 10 2>/dev/null | python -c "import json,sys;r=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$(basename $L)', round(r['keys_per_s']/1e9,3), 'G keys/s', round(r['tensor_frac'],3))"
  done
done
