mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_prefill_gpu.py tests/test_qjlc_gpu.py -x -q > gpurun_out/f2_gpu.log 2>&1; echo "exit $?" >> gpurun_out/f2_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/bench_f2.log 2>&1; echo "exit $?" >> gpurun_out/bench_f2.log
tail -15 gpurun_out/f2_gpu.log; grep '^{' gpurun_out/bench_f2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('prefill'))"; tail -3 gpurun_out/bench_f2.log
