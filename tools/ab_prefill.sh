#!/bin/bash
# A/B of the config-4 prefill (K1) across prebuilt libraries: tools/ab_prefill.sh libA.so libB.so [rounds]
R=${3:-2}
for r in $(seq $R); do
  for L in "$1" "$2"; do
    QJL_LIB=$L python tools/run_prefill.py 10 2>/dev/null | python -c "import json,sys;r=json.loads(sys.stdin.read().strip().splitlines()[-1]);p=r['parity'];print('$(basename $L)', round(r['keys_per_s']/1e9,3), 'G keys/s', round(r['kernel_ms']*1e3,1), 'us', round(r['tensor_frac_padded'],3), 'profile_us', round(r['with_profile']['ms']*1e3,1), 'flips', p['bit_flips_vs_fp64_kernel'], p['vs_oracle']['flips'], 'norms', p['fp16_norm_mismatches'])"
  done
done
