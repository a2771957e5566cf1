# F2: GPU tests, then C4 prefill numbers (K1 alone, profile + K1) for the shipped library and $1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for i in 1 2; do
for L in paper_2406_03482_b200/libqjl_b200.so $1; do
QJL_LIB=$L timeout 300 python tools/run_prefill.py 10 2>&1 | tail -1 | python -c "import json,sys;r=json.loads(sys.stdin.read());p=r['parity'];print('$(basename $L)', 'K1', round(r['kernel_ms']*1e3,1), 'us', round(r['keys_per_s']/1e9,3), 'Gk/s; prefill+profile', round(r['with_profile']['ms']*1e3,1), 'us', round(r['with_profile']['keys_per_s']/1e9,3), 'Gk/s; flips', p['bit_flips_vs_fp64_kernel'], p['vs_oracle']['flips'])"
done; done
