#!/bin/bash
# Round-2 evidence (one gpurun call, one GPU): bench lines of every config, the default
# bench run with cpu_baseline, the reference arm, ncu of the HBM-bound kernels at C3 / C5,
# and the in-sequence DRAM bytes per update of the unfused and fused passes.
cd "$(dirname "$0")/.."
TAG=${TAG:-r02}
O=gpurun_out
nproc; grep -m1 "model name" /proc/cpuinfo
# 1. default bench (C3, cpu_baseline with whole updates) and the reference arm
timeout 900 python bench.py > $O/bench_default_$TAG.json 2> $O/bench_default_$TAG.err; echo "default rc=$?"
timeout 1200 python bench.py --impl reference --steps 4 --warmup 1 > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err; echo "ref rc=$?"
# 2. every config
for c in 1 2 3 4 5; do
  st=16; [ $c = 5 ] && st=8
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu > $O/bench_c${c}_$TAG.json 2> $O/bench_c${c}_$TAG.err; echo "C$c rc=$?"
done
timeout 900 python bench.py --fused --steps 16 --warmup 3 --no-cpu > $O/bench_fused_$TAG.json 2> $O/bench_fused_$TAG.err; echo "fused rc=$?"
# 3. in-sequence DRAM bytes of every libsvd1 kernel, unfused and fused (C3, caches not flushed)
for f in "" "--fused"; do
  timeout 900 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
     -k 'regex:fmm_|secular|secfmm|loewner|colnorm|proj_|few_rows|householder|passthrough|col_rotate|probe|null_dir|gram_rows|thin_carry|apply_direct' --csv --log-file $O/dram_all${f}_$TAG.csv python bench.py $f --steps 2 --warmup 3 --no-e2e --no-check --no-cpu > /dev/null 2>&1; echo "dram$f rc=$?"
done
# 4. --set full of the HBM-bound kernels (projections, Householder, passthrough, few-rows) at C3 and C5
#    (HBM=0 skips it: gpurun brings back at most 64 MiB of gpurun_out/)
if [ "${HBM:-1}" != 0 ]; then
timeout 900 ncu --set full --clock-control none -k 'regex:proj_partial|proj_multi|householder|passthrough|few_rows|col_rotate|null_dir' -c 12 \
   -o $O/hbm_c3_$TAG -f python bench.py --steps 2 --warmup 1 --no-e2e --no-check --no-cpu > /dev/null 2>&1; echo "hbm c3 rc=$?"
timeout 1200 ncu --set full --clock-control none -k 'regex:proj_partial|householder|passthrough|few_rows' -c 10 \
   -o $O/hbm_c5_$TAG -f python bench.py --config 5 --steps 2 --warmup 1 --no-e2e --no-check --no-cpu > /dev/null 2>&1; echo "hbm c5 rc=$?"
fi
ls -la $O/*_$TAG*
