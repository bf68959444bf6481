#!/bin/bash
# Final evidence of a build (one gpurun call): default bench line, reference arm, every
# config's line, and the ncu launch list of the stream alone
cd "$(dirname "$0")/.."
TAG=${TAG:-r02b}
O=gpurun_out
nproc; grep -m1 "model name" /proc/cpuinfo
timeout 900 python bench.py > $O/bench_default_$TAG.json 2> $O/bench_default_$TAG.err; echo "default rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > $O/bench_2005_$TAG.json 2> $O/bench_2005_$TAG.err; echo "20/5 rc=$?"
timeout 1200 python bench.py --impl reference --steps 4 --warmup 1 > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err; echo "ref rc=$?"
for c in 1 2 4 5; do
  st=16; [ $c = 5 ] && st=8
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu > $O/bench_c${c}_$TAG.json 2> $O/bench_c${c}_$TAG.err; echo "C$c rc=$?"
done
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-check --no-cpu --no-seq"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$TAG.csv $CMD > /dev/null 2>&1; echo "launch list rc=$?"
ls -la $O/*_$TAG*
