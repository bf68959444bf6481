#!/bin/bash
# build variants of the few-rows kernel: its ncu time in the stream, batch parity, the C3 stream
cd "$(dirname "$0")/.."
for v in ${BVARS:-base}; do
  flags=$(echo $v | tr '~' ' '); [ "$v" = base ] && flags=""
  SVD1_NVCC_EXTRA="$flags" python paper_1707_08369_b200/build.py > gpurun_out/bv_build.log 2>&1 || { echo "build failed: $flags"; continue; }
  echo "== [$v]"
  python -m pytest tests/test_gpu_batch.py -x -q 2>&1 | tail -1
  timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active -k 'regex:few_rows' --csv \
    --log-file gpurun_out/few.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-check --no-cpu --no-seq > /dev/null 2>&1
  python tools/spec_summary.py gpurun_out/few.csv
  NREP=${NREP:-3} bash tools/gpu_var.sh 2>&1 | grep value
done
