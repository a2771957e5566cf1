# ncu --set full of the fused decode kernel (one launch) + summary
TAG=${1:-cur}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_udecode" -s 6 -c 1 -o gpurun_out/decode_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-prefill --no-extras > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu exit $?"
