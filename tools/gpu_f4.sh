mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_harness_gpu.py tests/test_prefill_gpu.py -x -q > gpurun_out/f4_gpu.log 2>&1; echo "exit $?" >> gpurun_out/f4_gpu.log
tail -25 gpurun_out/f4_gpu.log
