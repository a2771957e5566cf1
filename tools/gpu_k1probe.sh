# K1 ablations (1: no epilogue math, 2: no norm math, 3: both, 4: no MMA) + ncu of the shipped K1
for L in paper_2406_03482_b200/libqjl_b200.so variants/libqjl_k1a1.so variants/libqjl_k1a2.so variants/libqjl_k1a3.so variants/libqjl_k1a4.so; do
  QJL_LIB=$L timeout 300 python tools/run_prefill.py 10 2>/dev/null | python -c "import json,sys;r=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$(basename $L)', round(r['keys_per_s']/1e9,3), 'G keys/s', round(r['kernel_ms']*1e3,1), 'us', 'profile_us', round(r['with_profile']['ms']*1e3,1))"
done
timeout 300 python tools/run_prefill.py 3 > gpurun_out/plain_prefill.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quant_tc -s 2 -c 1 -o gpurun_out/quant_full python tools/run_prefill.py 3 > gpurun_out/ncu_full_q.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_detect -s 0 -c 2 -o gpurun_out/detect_full python tools/run_prefill.py 1 > gpurun_out/ncu_full_d.log 2>&1
tail -2 gpurun_out/ncu_full_q.log gpurun_out/ncu_full_d.log
