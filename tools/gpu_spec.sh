#!/bin/bash
# spectral kernel timings (ncu, gpu__time_duration + FP64 pipe) for env variants
cd "$(dirname "$0")/.."
for v0 in "X=1" ${VARS:-}; do v=$(echo $v0 | tr "~" " ");
  env $v timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
     -k 'regex:loewner|colnorm|secular_kernel|secfmm' --csv --log-file gpurun_out/spec_$v0.csv python tools/spectral_bench.py 4096 16384 > /dev/null 2>&1
  echo "== $v"; python tools/spec_summary.py gpurun_out/spec_$v0.csv
done
