set -x
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
bash tools/ab_prefill.sh variants/libqjl_k1old.so paper_2406_03482_b200/libqjl_b200.so 2 > gpurun_out/ab_k1.log 2>&1
cat gpurun_out/ab_k1.log
bash tools/ab.sh 3 variants/libqjl_mergeold.so paper_2406_03482_b200/libqjl_b200.so > gpurun_out/ab_merge.log 2>&1
cat gpurun_out/ab_merge.log
