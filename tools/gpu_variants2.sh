#!/bin/bash
# build variants of the GEMM kernel config and bench each (experiments)
cd "$(dirname "$0")/.."
for v in ${VARIANTS:-""}; do
  rm -f paper_1707_08369_b200/libsvd1.so
  SVD1_NVCC_EXTRA="$v" python paper_1707_08369_b200/build.py > gpurun_out/build_v.log 2>&1 || { echo "build failed $v"; continue; }
  for i in 1 2; do
    timeout 120 python bench.py --no-cpu --no-e2e --no-check > gpurun_out/bv.json 2>gpurun_out/bv.err
    echo "[$v] $(python tools/bench_brief.py gpurun_out/bv.json 2>&1 | cut -c1-130)"
  done
done
