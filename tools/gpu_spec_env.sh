#!/bin/bash
# environment variants (EVARS) of the spectral kernels: ncu durations at n = 4096, 16384 and the C3 stream
cd "$(dirname "$0")/.."
for e in ${EVARS:-X=1}; do
  echo "== $e"
  env $e timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
     -k 'regex:loewner|colnorm' --csv --log-file gpurun_out/spec_env.csv python tools/spectral_bench.py 4096 16384 > /dev/null 2>&1
  python tools/spec_summary.py gpurun_out/spec_env.csv
  NREP=${NREP:-2} ENVV=$e bash tools/gpu_var.sh 2>&1 | grep value
done
