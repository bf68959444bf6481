#!/bin/bash
# One gpurun call: every config's bench line, the C3 line with cpu baseline, the ncu
# launch list of a short C3 bench, and one ncu --set full capture of the FMM passes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/gpu_configs.sh
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-check --no-cpu"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fmm_gemm -s 192 -c 7 \
   -o gpurun_out/prof -f $CMD > gpurun_out/ncu.log 2>&1; echo "ncu full rc=$?"
