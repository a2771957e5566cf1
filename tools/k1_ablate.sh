for a in 0 1 2 3 4; do
  QJL_K1_ABLATE=$a python tools/run_prefill.py 10 2>/dev/null | python -c "import json,sys;r=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('ablate $a', round(r['keys_per_s']/1e9,3), 'G keys/s', round(r['kernel_ms']*1e3,1), 'us')"
done
