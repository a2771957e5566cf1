set -x
timeout 600 python -m pytest tests/test_decode_umma_gpu.py -x -q > gpurun_out/pytest_umma.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_umma.log
tail -15 gpurun_out/pytest_umma.log
timeout 300 python bench.py --no-cpu-baseline --no-prefill --steps 300 > gpurun_out/bench_umma.log 2>&1; echo "bench exit $?"
tail -2 gpurun_out/bench_umma.log | cut -c1-1500
