# small-batch decode: CTAs-per-unit caps (prebuilt variants) on C5 B1 / B4 points and C3
for pt in "--workload c5 --batch 1 --n 32768" "--workload c5 --batch 1 --n 131072" "--workload c5 --batch 4 --n 32768" "--workload c5 --batch 1 --n 4096" "--workload c3"; do
  AB_ARGS="$pt" bash tools/ab.sh 1 paper_2406_03482_b200/libqjl_b200.so "$@" | sed "s|^|$pt  |"
done
