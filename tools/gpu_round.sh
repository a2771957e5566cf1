# full round on one GPU: tests, smoke, bench (both arms), launch list, ncu of the top kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_[a-z]" -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_udecode -s 6 -c 1 -o gpurun_out/decode_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-prefill > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quant_tc -s 2 -c 1 -o gpurun_out/quant_full python tools/run_prefill.py 3 > gpurun_out/ncu_full_q.log 2>&1
timeout 600 ncu --section MemoryWorkloadAnalysis --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_udecode -s 6 -c 1 --csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-prefill > gpurun_out/ncu_traffic.csv 2>&1
ls -la gpurun_out
