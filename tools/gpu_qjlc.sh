mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_qjlc_gpu.py -x -q > gpurun_out/qjlc_gpu.log 2>&1; echo "exit $?" >> gpurun_out/qjlc_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/bench_q.log 2>&1; echo "exit $?" >> gpurun_out/bench_q.log
tail -30 gpurun_out/qjlc_gpu.log; grep '^{' gpurun_out/bench_q.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('qjlc'))"; tail -3 gpurun_out/bench_q.log
