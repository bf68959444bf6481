#!/bin/bash
# build variants of libsvd1 (compile-time knobs) and time the C3 stream with each
cd "$(dirname "$0")/.."
for v in ${BVARS}; do
  flags=$(echo $v | tr '~' ' ')
  SVD1_NVCC_EXTRA="$flags" python paper_1707_08369_b200/build.py > gpurun_out/bv_build.log 2>&1 || { echo "build failed: $flags"; tail -5 gpurun_out/bv_build.log; continue; }
  echo "== [$flags]"; NREP=${NREP:-3} bash tools/gpu_var.sh 2>&1 | grep value
done
