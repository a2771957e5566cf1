# C5 long-context sweep plus C2 full size: one bench.py line per point, each
# with the roofline object and the parity object (device decode vs the CPU oracle on as many
# whole units at full n as ~12 s of oracle work allows).  Output: gpurun_out/c5_sweep.jsonl
out=gpurun_out/c5_sweep.jsonl
: > $out
run() {
  timeout 600 python bench.py --no-prefill --steps 50 --warmup 5 "$@" > gpurun_out/sweep_one.log 2>&1
  rc=$?
  line=$(grep '^{' gpurun_out/sweep_one.log | tail -1)
  if [ -n "$line" ]; then echo "$line" >> $out; else echo "{\"args\": \"$*\", \"rc\": $rc, \"error\": \"no JSON line\"}" >> $out; tail -5 gpurun_out/sweep_one.log; fi
}
run --workload c2
for m in 256 512; do
  for n in 4096 32768 131072; do
    for b in 1 4 16 64; do
      run --workload c5 --batch $b --n $n --m-in $m
    done
  done
done
wc -l $out
