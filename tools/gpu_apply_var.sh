#!/bin/bash
# build variants (BVARS, '~' for spaces) x environment variants (EVARS): FMM-apply pass
# times alone, apply parity, C3 stream
cd "$(dirname "$0")/.."
for v in ${BVARS:-base}; do
  flags=$(echo $v | tr '~' ' '); [ "$v" = base ] && flags=""
  SVD1_NVCC_EXTRA="$flags" python paper_1707_08369_b200/build.py > gpurun_out/bv_build.log 2>&1 || { echo "build failed: $flags"; tail -5 gpurun_out/bv_build.log; continue; }
  python -m pytest tests/test_gpu_parity.py -x -q -k "cauchy or update_parity" 2>&1 | tail -1
  for e in ${EVARS:-X=1}; do
    echo "== [$v] [$e]"
    env $e SVD1_PASSTIME=1 python tools/apply_passes.py 4096 2>&1 | tail -2
    NREP=${NREP:-2} ENVV=$e bash tools/gpu_var.sh 2>&1 | grep value
  done
done
