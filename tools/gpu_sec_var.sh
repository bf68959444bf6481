#!/bin/bash
# secular-solve kernel variants: ncu time of the spectral kernels + parity + C3 stream
cd "$(dirname "$0")/.."
for v in ${BVARS}; do
  flags=$(echo $v | tr '~' ' ')
  SVD1_NVCC_EXTRA="$flags" python paper_1707_08369_b200/build.py > gpurun_out/bv_build.log 2>&1 || { echo "build failed: $flags"; tail -5 gpurun_out/bv_build.log; continue; }
  echo "== [$v]"
  python -m pytest tests/test_gpu_parity.py -x -q -k "secular" 2>&1 | tail -1
  timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
     -k 'regex:secular_kernel' --csv --log-file gpurun_out/sec.csv python tools/spectral_bench.py 4096 16384 > /dev/null 2>&1
  python tools/spec_summary.py gpurun_out/sec.csv
  NREP=${NREP:-2} bash tools/gpu_var.sh 2>&1 | grep value
done
