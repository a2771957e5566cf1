#!/bin/bash
# A/B benchmark of prebuilt libraries: tools/ab.sh ROUNDS lib1.so lib2.so ...
R=$1; shift
for r in $(seq $R); do
  for L in "$@"; do
    QJL_LIB=$L python bench.py --no-cpu-baseline --no-prefill --steps 300 ${AB_ARGS} 2>/dev/null | python -c "import json,sys;r=json.loads(sys.stdin.read().strip().splitlines()[-1]);s=r.get('scores_only') or {};print('$(basename $L)', 'step_us', round(r['ms_per_step']*1e3,1), 'kernel_us', round(r['roofline']['kernel_ms']*1e3,1), 'det_us', round((r['roofline'].get('deterministic_schedule_kernel_ms') or 0)*1e3,1), 'GB/s', round(r['value']), 'scores_us', round(s.get('ms_per_step',0)*1e3,1), r['clocks']['sm_mhz'])"
  done
done
