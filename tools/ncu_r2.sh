#!/bin/bash
# ncu evidence for round 2 (one gpurun call, one GPU, never multi-rank):
#  1. launch list (gpu__time_duration, clocks not locked) of the bench command -> per-kernel shares
#  2. --set full of 14 consecutive FMM GEMM passes inside the stream (two applies, U and V
#     sides, interleaved in launch order: per-apply figures are half the sums)
#  3. --set full of the spectral / HBM-bound kernels of one update (secular, Loewner, norms,
#     operator build, few-rows, projections, Householder, passthrough)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-check --no-cpu --no-seq"
TAG=${TAG:-r02}
timeout 300 $CMD > gpurun_out/ncu_plain_$TAG.json 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > /dev/null 2>&1; echo "launch list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:fmm_gemm -s ${GSKIP:-70} -c 14 \
   -o gpurun_out/gemm_$TAG -f $CMD > gpurun_out/ncu_gemm_$TAG.log 2>&1; echo "gemm capture rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on \
   -k 'regex:loewner|colnorm|secular_kernel|secfmm|fmm_ops|few_rows|proj_|householder|passthrough|col_rotate' -s ${SSKIP:-60} -c 24 \
   -o gpurun_out/spec_$TAG -f $CMD > gpurun_out/ncu_spec_$TAG.log 2>&1; echo "spectral capture rc=$?"
ls -la gpurun_out/*_$TAG*
